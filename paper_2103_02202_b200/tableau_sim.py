"""Native reference sample: the step before `sample_batch`.

Drop-in for `stabsim.tableau_sim.reference_sample(circuit, rng)`
(`stabsim/tableau_sim.py:326-329`): one noiseless run of the inverse-tableau
stabilizer simulator (SimState, tableau_sim.py:50-297), returning the
measurement record.  The simulator itself is C++ (`csrc/pfs_tableau.cpp`,
bit-packed tableau columns, phase-tracked Pauli products), reached through the
C-ABI `pfs_reference_sample`; it runs on the host and needs no GPU (SURVEY.md
§8(f) row 1: the reference takes ~35 min at d=100 in Python).

Randomness: each random measurement / reset collapse consumes one coin, in
circuit order — the reference draws `rng.integers(2)` there
(tableau_sim.py:177).  `reference_sample` draws its coin stream from `rng` up
front; `reference_sample_with_coins` takes an explicit stream (the parity
tests feed the reference and this simulator the same coins).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .circuit import as_circuit, iter_flat

# gate codes of include/pfs.h (enum pfs_tableau_gate)
GATE_CODES = {"I": 0, "X": 1, "Y": 2, "Z": 3, "H": 4, "S": 5, "S_DAG": 6, "SQRT_X": 7,
              "SQRT_X_DAG": 8, "SQRT_Y": 9, "SQRT_Y_DAG": 10, "CNOT": 11, "CY": 12, "CZ": 13,
              "SWAP": 14, "M": 15, "R": 16, "MR": 17}
COLLAPSING = ("M", "R", "MR")


def lower(circuit):
    """(ops int32 [n, 3] = (gate code, n_targets, target offset), targets,
    num_qubits, num_measurements, collapsing targets); noise channels and
    annotations carry no effect on a noiseless run and are dropped."""
    c = as_circuit(circuit)
    ops, targets = [], []
    n_coll = 0
    for ins in iter_flat(c):
        code = GATE_CODES.get(ins.gate.name)
        if code is None:
            continue
        ops.append((code, len(ins.targets), len(targets)))
        targets.extend(int(t) for t in ins.targets)
        if ins.gate.name in COLLAPSING:
            n_coll += len(ins.targets)
    ops_a = np.asarray(ops, dtype=np.int32).reshape(-1, 3)
    return ops_a, np.asarray(targets, dtype=np.int32), c.num_qubits, c.num_measurements, n_coll


def reference_sample_with_coins(circuit, coins, lowered=None) -> tuple[np.ndarray, np.ndarray, int]:
    """(measurement bits uint8, determined flags uint8, random measurements)."""
    ops, tg, nq, nm, _ = lowered if lowered is not None else lower(circuit)
    coins = np.ascontiguousarray(np.asarray(coins, dtype=np.uint8).reshape(-1))
    bits = np.zeros(max(nm, 1), dtype=np.uint8)
    det = np.zeros(max(nm, 1), dtype=np.uint8)
    written = ctypes.c_int64(0)
    L = N.lib()
    P = N._p
    rc = L.pfs_reference_sample(P(ops), ops.shape[0], P(tg), tg.shape[0], nq, P(coins),
                                coins.shape[0], P(bits), P(det), nm, ctypes.byref(written))
    if rc != 0:
        msg = L.pfs_reference_sample_error().decode(errors="replace")
        raise (ValueError if rc == N.E_INVALID else RuntimeError)(msg)
    if written.value != nm:
        raise RuntimeError(f"reference sample wrote {written.value} of {nm} measurements")
    used = int(np.count_nonzero(det[:nm] == 0))  # random measurements (resets may add more)
    return bits[:nm], det[:nm], used


def reference_sample(circuit, rng=None) -> list[int]:
    """One noiseless sample of the circuit's measurement record
    (stabsim/tableau_sim.py:326-329)."""
    lowered = lower(circuit)
    if rng is None or isinstance(rng, (int, np.integer)):
        rng = np.random.default_rng(rng)
    coins = rng.integers(0, 2, size=max(lowered[4], 1), dtype=np.uint8)
    bits, _, _ = reference_sample_with_coins(circuit, coins, lowered)
    return [int(b) for b in bits]
