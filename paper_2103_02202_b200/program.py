"""Flat frame program: the circuit lowered to a flat instruction table.

This is the B200 build's counterpart of `compile_frame_program`
(`stabsim/frame_sim.py:170-189`): REPEAT is expanded (`iter_flat`,
circuit.py:100-107), Pauli gates and I are dropped (empty frame plan,
frame_sim.py:176-178), every other instruction becomes one row of an int32
table.  Unlike the reference's tuple list it also numbers, once and for all,

* measurement records (flat order, targets left to right — frame_sim.py:183-186),
* coin rows: qubit init rows 0..n-1, then per collapsing target M/R -> 1,
  MR -> 2 (the row numbering of the reference's `rng.bytes()` calls,
  SURVEY.md Appendix E),
* noise mask rows: per noise instruction, per target, x row then z row,
* noise instruction ordinals (the Philox counter domain),

so the CUDA kernels, the C oracle and the injected-mask harness all address
the same random streams.  Detectors and observables are kept as record-index
sets (CSR) in output-column order: detectors, then observables.

Instruction row layout (int32 x 8):
    0 kind   1 code   2 n_targets   3 tgt_off   4 rec_base   5 coin_base
    6 noise_row_base   7 aux (noise ordinal | detector/observable column)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import gates as G
from .circuit import as_circuit, _is_repeat

K_GATE, K_M, K_R, K_MR, K_NOISE, K_DET, K_OBS = range(7)
CH_XERR, CH_YERR, CH_ZERR, CH_DEP1, CH_DEP2 = range(5)
_CHANNEL = {"X_ERROR": CH_XERR, "Y_ERROR": CH_YERR, "Z_ERROR": CH_ZERR,
            "DEPOLARIZE1": CH_DEP1, "DEPOLARIZE2": CH_DEP2}
CHANNEL_ARITY = {CH_XERR: 1, CH_YERR: 1, CH_ZERR: 1, CH_DEP1: 1, CH_DEP2: 2}
CHANNEL_PATTERNS = {
    CH_XERR: G.GATE_MAP["X_ERROR"].noise_patterns,
    CH_YERR: G.GATE_MAP["Y_ERROR"].noise_patterns,
    CH_ZERR: G.GATE_MAP["Z_ERROR"].noise_patterns,
    CH_DEP1: G.GATE_MAP["DEPOLARIZE1"].noise_patterns,
    CH_DEP2: G.GATE_MAP["DEPOLARIZE2"].noise_patterns,
}
RULE_ARITY = {G.RULE_SWAPXZ: 1, G.RULE_ZXORX: 1, G.RULE_XXORZ: 1, G.RULE_CX: 2,
              G.RULE_CZ: 2, G.RULE_CY: 2, G.RULE_SWAP: 2}

# Frame bits read+written per shot for collapses.
_COLLAPSE_BITS = {K_M: 4, K_R: 2, K_MR: 4}


@dataclass
class FlatProgram:
    num_qubits: int
    num_measurements: int
    num_detectors: int
    num_observables: int
    instrs: np.ndarray      # int32 [n, 8]
    targets: np.ndarray     # int32
    noise_p: np.ndarray     # float64 [n_noise]
    det_ptr: np.ndarray     # int64 [num_columns + 1]
    det_idx: np.ndarray     # int64 absolute record indices
    num_coin_rows: int
    num_noise_rows: int
    bframe_bits: int        # algorithmic frame bits per shot

    @property
    def num_columns(self) -> int:
        return self.num_detectors + self.num_observables

    @property
    def num_noise(self) -> int:
        return int(self.noise_p.shape[0])

    def counts(self) -> dict:
        k = self.instrs[:, 0]
        return {"instrs": int(self.instrs.shape[0]), "gates": int((k == K_GATE).sum()),
                "collapses": int(np.isin(k, (K_M, K_R, K_MR)).sum()),
                "noise": int((k == K_NOISE).sum())}


def flatten(circuit) -> FlatProgram:
    """Lower a circuit (text, ours, or a reference Circuit) to a FlatProgram."""
    c = as_circuit(circuit)
    rows: list[tuple] = []
    targets: list[int] = []
    noise_p: list[float] = []
    det_sets: list[list[int]] = []
    obs_acc: dict[int, dict[int, int]] = {}
    obs_events: list[tuple[int, list[int]]] = []
    state = {"rec": 0, "coin": c.num_qubits, "nrow": 0, "bits": 0}

    def emit(elements):
        for e in elements:
            if _is_repeat(e):
                for _ in range(e.count):
                    emit(e.body.elements)
                continue
            g = e.gate
            if g.kind == G.UNITARY:
                if g.rule == G.RULE_NONE:
                    continue
                off = len(targets)
                targets.extend(e.targets)
                rows.append((K_GATE, g.rule, len(e.targets), off, 0, 0, 0, 0))
                state["bits"] += G.RULE_BITS[g.rule] * (len(e.targets) // g.arity)
            elif g.kind == G.COLLAPSING:
                kind = K_MR if (g.records and g.resets) else (K_M if g.records else K_R)
                off = len(targets)
                targets.extend(e.targets)
                n = len(e.targets)
                rows.append((kind, 0, n, off, state["rec"], state["coin"], 0, 0))
                if g.records:
                    state["rec"] += n
                state["coin"] += n * (2 if kind == K_MR else 1)
                state["bits"] += _COLLAPSE_BITS[kind] * n
            elif g.kind == G.NOISE:
                off = len(targets)
                targets.extend(e.targets)
                n = len(e.targets)
                if e.param is None:
                    raise ValueError(f"{g.name} needs a parameter")
                rows.append((K_NOISE, _CHANNEL[g.name], n, off, 0, 0, state["nrow"],
                             len(noise_p)))
                noise_p.append(float(e.param))
                state["nrow"] += 2 * n
            elif g.name == "DETECTOR":
                d = len(det_sets)
                det_sets.append([state["rec"] + k for k in e.targets])
                rows.append((K_DET, 0, 0, 0, 0, 0, 0, d))
            elif g.name == "OBSERVABLE_INCLUDE":
                k = int(e.param)
                acc = obs_acc.setdefault(k, {})
                recs = [state["rec"] + t for t in e.targets]
                for m in recs:
                    acc[m] = acc.get(m, 0) ^ 1
                obs_events.append((k, recs))
                off = len(targets)
                targets.extend(recs)
                rows.append((K_OBS, 0, len(recs), off, 0, 0, 0, k))
            # TICK: nothing

    emit(c.elements)
    num_det = len(det_sets)
    num_obs = (max(obs_acc) + 1) if obs_acc else 0
    cols = det_sets + [sorted(m for m, v in obs_acc.get(i, {}).items() if v)
                       for i in range(num_obs)]
    ptr = np.zeros(len(cols) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(s) for s in cols])
    idx = np.fromiter((m for s in cols for m in s), dtype=np.int64, count=int(ptr[-1]))
    instrs = np.array(rows, dtype=np.int32).reshape(-1, 8)
    # observable rows carry the final column index in aux
    if num_obs:
        sel = instrs[:, 0] == K_OBS
        instrs[sel, 7] += num_det
    return FlatProgram(
        num_qubits=c.num_qubits, num_measurements=state["rec"], num_detectors=num_det,
        num_observables=num_obs, instrs=instrs,
        targets=np.array(targets, dtype=np.int32), noise_p=np.array(noise_p, dtype=np.float64),
        det_ptr=ptr, det_idx=idx, num_coin_rows=state["coin"], num_noise_rows=state["nrow"],
        bframe_bits=state["bits"])
