"""Shared helpers for the parity tests."""

from __future__ import annotations

import glob
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def inject_cases():
    return sorted(os.path.basename(f)[7:-4] for f in glob.glob(os.path.join(GOLDEN, "inject_*.npz")))


def load_inject(name):
    from oracle.inject import make_streams

    z = np.load(os.path.join(GOLDEN, f"inject_{name}.npz"))
    text = str(z["text"])
    B = int(z["B"])
    coins, masks = make_streams(text, B, int(z["seed"]), int(z["density_k"]))
    return text, B, coins, masks, z["flips_b8"], z["events_b8"]


def load_stats(name):
    z = np.load(os.path.join(GOLDEN, f"stats_{name}.npz"))
    return str(z["text"]), int(z["shots"]), z["counts"], z["pairs"], z["pair_counts"]


def load_noiseless(name):
    z = np.load(os.path.join(GOLDEN, f"noiseless_{name}.npz"))
    return str(z["text"]), z["reference"], z["deterministic"]


def load_exact():
    with open(os.path.join(GOLDEN, "exact_tiny.json")) as f:
        return json.load(f)


def b8_unpack(b8: np.ndarray, num_results: int) -> np.ndarray:
    return np.unpackbits(b8, axis=1, bitorder="little")[:, :num_results]


def rows_unpack(rows: np.ndarray, num_shots: int) -> np.ndarray:
    """uint32 rows [R, words] -> uint8 [shots, R]."""
    by = np.ascontiguousarray(rows).view(np.uint8)
    bits = np.unpackbits(by, axis=1, bitorder="little")[:, :num_shots]
    return np.ascontiguousarray(bits.T)


def five_sigma(count_a, n_a, count_b, n_b, sigmas=5.0):
    """Max |z| of per-column binomial frequency differences."""
    fa = np.asarray(count_a, dtype=np.float64) / n_a
    fb = np.asarray(count_b, dtype=np.float64) / n_b
    f = (np.asarray(count_a, dtype=np.float64) + count_b) / (n_a + n_b)
    sd = np.sqrt(np.maximum(f * (1 - f), 1.0 / (n_a + n_b)) * (1.0 / n_a + 1.0 / n_b))
    z = np.abs(fa - fb) / sd
    return float(z.max()) if z.size else 0.0


def pair_counts(bits: np.ndarray, pairs: np.ndarray) -> np.ndarray:
    b = bits.astype(np.int64)
    return (b[:, pairs[:, 0]] & b[:, pairs[:, 1]]).sum(axis=0)
