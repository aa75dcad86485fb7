"""Injected-mask streams — TEST INFRASTRUCTURE.

This module is part of the parity oracle: only tests/, `__graft_entry__.smoke()`
and bench.py's CPU-baseline leg may import it.  It builds the seeded
coin / noise-mask rows that drive the reference's own `FrameBatch`
(tests/golden/make_golden.py), the C oracle and the CUDA injected mode with
identical bits.

Row layout: uint32 [rows, words], shot s of a row = bit (s & 31) of word
(s >> 5) — the little-endian byte order of `BitBuffer.to_bytes()`
(`stabsim/bitvec.py:50-52`).

* coin rows, in the reference's `rng.bytes()` call order: one per qubit
  (`FrameBatch.__init__`, frame_sim.py:38-39), then per collapsing target in
  flat order M -> 1 (frame_sim.py:79), R -> 1 (frame_sim.py:85),
  MR -> 2 (measure's, then reset's; frame_sim.py:87-90).
* noise rows: per noise instruction in flat order, per target: x-mask row then
  z-mask row (DEPOLARIZE2: per pair, slot 0 then slot 1).
"""

from __future__ import annotations

import numpy as np


def stream_sizes(circuit) -> tuple[int, int]:
    """(coin rows, noise rows) of a circuit (our Circuit or duck-typed)."""
    from paper_2103_02202_b200.circuit import as_circuit, iter_flat

    c = as_circuit(circuit)
    coins = c.num_qubits
    noise = 0
    for ins in iter_flat(c):
        g = ins.gate
        if g.kind == "collapsing":
            coins += len(ins.targets) * (2 if (g.records and g.resets) else 1)
        elif g.kind == "noise":
            noise += 2 * len(ins.targets)
    return coins, noise


def random_rows(seed: int, n_rows: int, n_bits: int, density_k: int = 1) -> np.ndarray:
    """uint32 [n_rows, ceil(n_bits/64)*2] rows of Bernoulli(2^-k) bits.

    Drawn from PCG64.random_raw (a stable raw bit stream); bits at or past
    n_bits are zero.
    """
    w64 = (n_bits + 63) // 64
    bg = np.random.PCG64(seed)
    out = np.full((n_rows, w64), np.uint64(0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
    for _ in range(max(1, density_k)):
        out &= bg.random_raw(n_rows * w64).astype(np.uint64).reshape(n_rows, w64)
    rem = n_bits % 64
    if rem and w64:
        out[:, -1] &= np.uint64((1 << rem) - 1)
    return out.view(np.uint32).reshape(n_rows, 2 * w64)


def zero_channel_rows(circuit, noise_rows: np.ndarray) -> np.ndarray:
    """Zero mask rows a channel cannot touch (z for X_ERROR, x for Z_ERROR),
    keeping channel realism (Appendix E); both engines accept any mask."""
    from paper_2103_02202_b200.circuit import as_circuit, iter_flat

    c = as_circuit(circuit)
    out = noise_rows.copy()
    r = 0
    for ins in iter_flat(c):
        if ins.gate.kind != "noise":
            continue
        name = ins.gate.name
        for _t in ins.targets:
            if name == "X_ERROR":
                out[r + 1] = 0
            elif name == "Z_ERROR":
                out[r] = 0
            r += 2
    return out


def make_streams(circuit, n_bits: int, seed: int, density_k: int):
    """(coins, noise) uint32 row arrays for a circuit and shot count."""
    n_coin, n_noise = stream_sizes(circuit)
    coins = random_rows(seed, n_coin, n_bits, 1)
    noise = random_rows(seed + 1, n_noise, n_bits, density_k)
    noise = zero_channel_rows(circuit, noise)
    return coins, noise
