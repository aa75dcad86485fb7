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


# ---------------------------------------------------------------- RNG layout
def rule_chunk_length(p: float, apps: int, tile_shots: int, target: float) -> int:
    """the power of two nearest (in ratio) to target / p trials,
    halved while half of it still covers the instruction's trials (p == 1:
    up to 1024, p == 0: 1)."""
    N = apps * tile_shots
    L = 1
    if N == 0 or p <= 0.0:
        return L
    if p >= 1.0:
        while L < N and L < 1024:
            L *= 2
        return L
    want = target / p
    while L * 2 <= want * 1.41421356 and L < (1 << 27):
        L *= 2
    while L > 1 and L // 2 >= N:
        L //= 2
    return L


def rule_chunk_lengths(prog, tile_shots: int, target: float = 2.0) -> np.ndarray:
    """Chunk length of every noise instruction of a FlatProgram by the rule."""
    out = np.ones(prog.num_noise, dtype=np.uint32)
    for row in prog.instrs:
        if row[0] == 4:  # K_NOISE
            ar = 2 if row[1] == 4 else 1
            out[row[7]] = rule_chunk_length(float(prog.noise_p[row[7]]), int(row[2]) // ar, tile_shots, target)
    return out


def product_layout(sampler):
    """(T, S, chunk_L): the RNG layout a compiled sampler draws with."""
    params, _ = sampler.native.noise_schedule()
    T = sampler.tile_shots
    S = 32 if sampler.native.info["kernel"] == 4 else 32 * min(T // 32, 4)
    return T, S, params[:, 0].copy()


def oracle_run(oracle, sampler, shots: int, seed: int, shot_offset: int = 0, **kw):
    """The oracle's draws with the sampler's layout: (flip rows, event rows)."""
    T, S, L = product_layout(sampler)
    assert shot_offset % T == 0
    return oracle.sample(sampler.flat, shots, T, seed=seed, tile_offset=shot_offset // T, chunk_L=L,
                         vector_shots=S, **kw)
