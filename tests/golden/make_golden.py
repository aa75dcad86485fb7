"""Generate the golden fixtures by running the REFERENCE itself.

Runs only in the build container, where the reference package is mounted at
/root/reference (it does not travel to the GPU box); the outputs are the
committed files next to this script.  Usage:

    python tests/golden/make_golden.py            # all fixtures

Fixtures (all derived from `stabsim` at /root/reference/pkg/src):

* frame_plans.json   — `GateData.frame_plan` / `noise_patterns` per gate
                        (stabsim/gates.py:70-92, 354-360).
* inject_*.npz       — (T2) injected-mask runs of the reference's own
                        `FrameBatch` opcode loop (frame_sim.py:192-205) with
                        the coin stream fed through `.bytes()` and opcode 4
                        replaced by XOR of supplied mask rows.
                        Stores circuit text, B, seed, density, flips and events
                        (b8, shot-major) — masks are regenerated from the seed
                        by oracle/inject.py.
* noiseless_*.npz    — (T1) `tableau_sim.reference_sample` + which records are
                        deterministic (flip 0 under two coin streams).
* stats_*.npz        — (T3) per-detector and pairwise event counts from
                        `collect_flips` + `detector_events` (reference RNG).
* exact_*.json       — `oracle.enumerate_distribution` of tiny noisy circuits
                        with the reference sample used to sample them.
* refsample_*.npz    — `tableau_sim.SimState.run(skip_noise=True)` (the body of
                        `reference_sample`, tableau_sim.py:326-329) driven by a
                        supplied collapse-coin stream: circuit text, coins,
                        measurement bits and `determined_record`.
"""

from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REPO)
sys.path.insert(0, REF_SRC)

from oracle.inject import make_streams  # noqa: E402
from paper_2103_02202_b200 import circuit as mc  # noqa: E402
from paper_2103_02202_b200 import generators as gen  # noqa: E402


def _ref():
    from stabsim import bitvec, circuit, frame_sim, gates, io_formats, oracle, tableau_sim
    return bitvec, circuit, frame_sim, gates, io_formats, oracle, tableau_sim


class _RowStream:
    """Stands in for the numpy Generator: `.bytes(n)` returns the next row."""

    def __init__(self, rows: np.ndarray, nbytes: int):
        self.rows = rows
        self.nbytes = nbytes
        self.k = 0

    def bytes(self, n):
        assert n == self.nbytes, (n, self.nbytes)
        row = self.rows[self.k]
        self.k += 1
        return row.tobytes()[:n]


def run_reference_injected(text: str, B: int, coins: np.ndarray, noise: np.ndarray):
    """Drive the reference FrameBatch with injected coins and noise masks."""
    bitvec, rcircuit, frame_sim, gates, io_formats, _, _ = _ref()
    rc = rcircuit.parse(mc.to_reference_dialect(text))
    program = frame_sim.compile_frame_program(rc)
    assert B % 64 == 0
    stream = _RowStream(coins, B // 8)
    batch = frame_sim.FrameBatch(rc.num_qubits, B, stream)
    nr = 0
    for op in program:
        kind = op[0]
        if kind == 0:
            for app in op[2]:
                batch._apply_plan(op[1], app)
        elif kind == 1:
            batch.measure(op[1])
        elif kind == 2:
            batch.reset(op[1])
        elif kind == 3:
            batch.measure_reset(op[1])
        else:
            _, gate, _p, targets = op
            for t in targets:
                xm = int.from_bytes(noise[nr].tobytes()[:B // 8], "little")
                zm = int.from_bytes(noise[nr + 1].tobytes()[:B // 8], "little")
                batch.x_table.rows[t].bits ^= xm
                batch.z_table.rows[t].bits ^= zm
                nr += 2
    assert stream.k == coins.shape[0], (stream.k, coins.shape)
    assert nr == noise.shape[0]
    M = rc.num_measurements
    table = bitvec.BitTable(len(batch.flip_rows), batch.batch_size, batch.flip_rows)
    rows = frame_sim._transpose_flips(table, M)
    flips = io_formats.SampleTable.from_rows(rows, M)
    events = io_formats.detector_events(flips, rcircuit.detector_sets(rc))
    return _b8(io_formats, flips), _b8(io_formats, events)


def _b8(io_formats, table):
    nb = (table.num_results + 7) // 8
    raw = io_formats.write_b8(table)
    return np.frombuffer(raw, dtype=np.uint8).reshape(table.num_shots, nb).copy()


def mixed_circuit(seed: int, n: int, n_instr: int, noise_p=(0.05, 0.2)) -> str:
    """Small random circuit using every gate kind, duplicate targets, conflicts
    inside one instruction (`CX 0 1 1 2`), REPEAT, detectors and observables."""
    rng = np.random.default_rng(seed)
    one = ["I", "X", "Y", "Z", "H", "S", "S_DAG", "SQRT_Y", "SQRT_Y_DAG", "SQRT_X",
           "SQRT_X_DAG"]
    two = ["CX", "CY", "CZ", "SWAP", "CNOT"]
    noise1 = ["X_ERROR", "Y_ERROR", "Z_ERROR", "DEPOLARIZE1"]
    lines = []
    meas = 0

    def body(count):
        nonlocal meas
        out = []
        for _ in range(count):
            r = rng.random()
            if r < 0.25:
                g = one[rng.integers(len(one))]
                k = int(rng.integers(1, n + 2))
                ts = rng.integers(0, n, size=k)  # duplicates allowed
                out.append(f"{g} " + " ".join(map(str, ts)))
            elif r < 0.5:
                g = two[rng.integers(len(two))]
                k = int(rng.integers(1, n))
                ts = []
                for _ in range(k):
                    a, b = rng.choice(n, size=2, replace=False)
                    ts += [int(a), int(b)]
                out.append(f"{g} " + " ".join(map(str, ts)))
            elif r < 0.68:
                g = ["M", "R", "MR"][rng.integers(3)]
                k = int(rng.integers(1, n + 1))
                ts = rng.integers(0, n, size=k)
                out.append(f"{g} " + " ".join(map(str, ts)))
                if g != "R":
                    meas += k
            elif r < 0.85:
                p = float(rng.choice(noise_p))
                if rng.random() < 0.7:
                    g = noise1[rng.integers(len(noise1))]
                    k = int(rng.integers(1, n + 2))
                    ts = rng.integers(0, n, size=k)
                else:
                    g = "DEPOLARIZE2"
                    k = int(rng.integers(1, n))
                    ts = []
                    for _ in range(k):
                        a, b = rng.choice(n, size=2, replace=False)
                        ts += [int(a), int(b)]
                out.append(f"{g}({p}) " + " ".join(map(str, ts)))
            elif r < 0.95:
                if meas:
                    k = int(rng.integers(1, min(4, meas) + 1))
                    lb = rng.choice(min(meas, 12), size=k, replace=False) + 1
                    out.append("DETECTOR " + " ".join(f"rec[-{int(v)}]" for v in lb))
            else:
                if meas:
                    lb = int(rng.integers(1, min(meas, 6) + 1))
                    out.append(f"OBSERVABLE_INCLUDE({int(rng.integers(2))}) rec[-{lb}]")
                else:
                    out.append("TICK")
        return out

    # make sure every qubit index appears so num_qubits == n
    lines.append("R " + " ".join(map(str, range(n))))
    lines += body(n_instr // 2)
    rep = body(max(2, n_instr // 4))
    # REPEAT body must only look back within what exists at first iteration:
    lines.append("REPEAT 3 {")
    lines += ["    " + s for s in rep]
    lines.append("}")
    lines += body(n_instr // 4)
    lines.append("M " + " ".join(map(str, range(n))))
    lines.append(f"DETECTOR rec[-1] rec[-{n}]")
    lines.append("OBSERVABLE_INCLUDE(0) rec[-2]")
    lines.append("OBSERVABLE_INCLUDE(1) rec[-3]")
    return "\n".join(lines) + "\n"


def valid(text):
    try:
        c = mc.parse(text)
        mc.to_reference_dialect(c)
        return True
    except Exception:
        return False


INJECT_CASES = [
    # name, text factory, B, seed, density k
    ("c0_d3", lambda: gen.surface_code_memory(3, 3, 1e-3), 1024, 11, 5),
    ("d5", lambda: gen.surface_code_memory(5, 5, 5e-3), 1024, 12, 5),
    ("c1_random", lambda: gen.random_clifford(64, 200, 0.01, 0), 1024, 13, 8),
    ("d7_flat", lambda: gen.surface_code_memory(7, 3, 1e-3, use_repeat=False), 256, 14, 4),
]


def mixed_cases():
    out = []
    seed = 100
    while len(out) < 10:
        n = [3, 5, 8, 12, 33, 70][len(out) % 6]
        t = mixed_circuit(seed, n, 40 + 4 * len(out))
        seed += 1
        if valid(t):
            B = [64, 192, 128, 320, 64, 256, 1024, 64, 192, 128][len(out)]
            out.append((f"mix{len(out)}", t, B, 200 + len(out), 2 + len(out) % 3))
    return out


def gen_inject():
    cases = [(n, f(), B, s, k) for n, f, B, s, k in INJECT_CASES] + mixed_cases()
    for name, text, B, seed, k in cases:
        t0 = time.time()
        coins, noise = make_streams(text, B, seed, k)
        flips, events = run_reference_injected(text, B, coins, noise)
        np.savez_compressed(os.path.join(HERE, f"inject_{name}.npz"),
                            text=np.array(text), B=B, seed=seed, density_k=k,
                            flips_b8=flips, events_b8=events)
        print(f"inject {name}: B={B} flips={flips.shape} events={events.shape} "
              f"{time.time() - t0:.1f}s", flush=True)


def gen_frame_plans():
    _, _, _, gates, _, _, _ = _ref()
    out = {}
    for g in gates.GATES:
        rec = {"kind": g.kind, "arity": g.arity}
        if g.kind == gates.UNITARY:
            rec["frame_plan"] = [[p, s, [list(x) for x in src]] for p, s, src in g.frame_plan]
        if g.kind == gates.NOISE:
            rec["noise_patterns"] = [list(p) for p in g.noise_patterns]
        rec["records"] = g.records
        rec["resets"] = g.resets
        out[g.name] = rec
    with open(os.path.join(HERE, "frame_plans.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("frame_plans.json", len(out))


def gen_noiseless():
    bitvec, rcircuit, frame_sim, gates, io_formats, _, tableau_sim = _ref()
    cases = [("d3", gen.surface_code_memory(3, 3, 0.0)),
             ("d5", gen.surface_code_memory(5, 5, 0.0)),
             ("c1", gen.random_clifford(64, 200, 0.0, 0)),
             ("mix", mixed_circuit(7, 6, 50, noise_p=(0.0,)))]
    for name, text in cases:
        rc = rcircuit.parse(mc.to_reference_dialect(text))
        ref = tableau_sim.reference_sample(rc, np.random.default_rng(5))
        det = np.ones(rc.num_measurements, dtype=bool)
        for s in (1, 2):
            fl = frame_sim.collect_flips(rc, 1024, np.random.default_rng(s)).to_numpy()
            det &= ~fl.any(axis=0)
        np.savez_compressed(os.path.join(HERE, f"noiseless_{name}.npz"), text=np.array(text),
                            reference=np.array(ref, dtype=np.uint8), deterministic=det)
        print(f"noiseless {name}: M={rc.num_measurements} det={int(det.sum())}", flush=True)


def _stat_worker(args):
    text, shots, seed, B, pairs = args
    _, rcircuit, frame_sim, _, io_formats, _, _ = _ref()
    rc = rcircuit.parse(mc.to_reference_dialect(text))
    fl = frame_sim.collect_flips(rc, shots, np.random.default_rng(seed), B)
    ev = io_formats.detector_events(fl, rcircuit.detector_sets(rc)).to_numpy().astype(np.uint8)
    del fl
    counts = ev.sum(axis=0, dtype=np.int64)
    pc = np.zeros(len(pairs), dtype=np.int64)
    for i in range(0, len(pairs), 1024):  # bounded temporaries (d=25: 16k columns)
        pp = pairs[i:i + 1024]
        pc[i:i + 1024] = (ev[:, pp[:, 0]] & ev[:, pp[:, 1]]).sum(axis=0, dtype=np.int64)
    return counts, pc


def make_pairs(num_det: int, per_round: int, seed: int, n_random: int = 4000):
    rng = np.random.default_rng(seed)
    pairs = []
    for s in sorted({1, 2, per_round} - {0}):
        pairs += [(i, i + s) for i in range(num_det - s)]
    a = rng.integers(0, num_det, size=n_random)
    b = rng.integers(0, num_det, size=n_random)
    pairs += [(int(x), int(y)) for x, y in zip(a, b) if x != y]
    return np.array(pairs, dtype=np.int64).reshape(-1, 2)


def _stat_subprocess(job):
    """Run one stats shard in a fresh interpreter (fork/spawn pools hang here)."""
    import pickle
    import subprocess
    import tempfile

    with tempfile.NamedTemporaryFile(suffix=".pkl", delete=False) as f:
        pickle.dump(job, f)
        path = f.name
    subprocess.run([sys.executable, os.path.abspath(__file__), "_statjob", path], check=True)
    with open(path + ".out", "rb") as f:
        return pickle.load(f)


def gen_stats(procs: int, only=None):
    cases = [
        ("d3", gen.surface_code_memory(3, 3, 1e-2), 1 << 16, 1024, 8),
        ("d5", gen.surface_code_memory(5, 5, 5e-3), 1 << 16, 4096, 24),
        ("c1", gen.random_clifford(64, 200, 0.01, 0), 1 << 15, 1024, 6),
        ("d25", gen.surface_code_memory(25, 25, 1e-3), 1 << 20, 8192, 624),
    ]
    for name, text, shots, B, per_round in cases:
        if only and name not in only:
            continue
        t0 = time.time()
        c = mc.parse(text)
        nd = len(mc.detector_and_observable_sets(c))
        pairs = make_pairs(nd, per_round, 3)
        # shards of at most 8192 shots keep each worker's event matrix small
        n_jobs = max(procs, shots // 8192)
        per = shots // n_jobs
        jobs = [(text, per, 1000 + i, B, pairs) for i in range(n_jobs)]
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(procs) as pool:
            res = list(pool.map(_stat_subprocess, jobs))
        counts = sum(r[0] for r in res)
        pc = sum(r[1] for r in res)
        np.savez_compressed(os.path.join(HERE, f"stats_{name}.npz"), text=np.array(text),
                            shots=per * n_jobs, counts=counts, pairs=pairs, pair_counts=pc)
        print(f"stats {name}: shots={per * n_jobs} det={nd} mean rate="
              f"{counts.mean() / (per * n_jobs):.4g} {time.time() - t0:.1f}s", flush=True)


TINY = [
    "R 0 1\nH 0\nCX 0 1\nDEPOLARIZE2(0.1) 0 1\nM 0 1\n",
    "H 0\nS 0\nX_ERROR(0.2) 0\nM 0\nMR 0\nY_ERROR(0.3) 0\nM 0\n",
    "R 0 1 2\nH 1\nCY 1 2\nSWAP 0 1\nDEPOLARIZE1(0.25) 0 1 2\nCZ 0 2\nSQRT_Y 2\nM 0 1 2\n",
    "H 0 1\nCX 0 2 1 3\nZ_ERROR(0.15) 0\nH 0\nM 0 1\nDEPOLARIZE2(0.2) 2 3\nM 2 3\nR 0\nM 0\n",
    "R 0 1 2 3\nSQRT_X 0\nS_DAG 1\nCX 0 1\nSQRT_Y_DAG 2\nCZ 2 3\nX_ERROR(0.4) 3\nMR 0 1\nH 0\nM 0 2 3\n",
]


def gen_exact():
    _, rcircuit, _, _, _, oracle, tableau_sim = _ref()
    out = []
    for text in TINY:
        rc = rcircuit.parse(mc.to_reference_dialect(text))
        dist = oracle.enumerate_distribution(rc)
        ref = tableau_sim.reference_sample(rc, np.random.default_rng(9))
        out.append({"text": text, "reference": list(map(int, ref)),
                    "dist": [[list(k), v] for k, v in sorted(dist.items())]})
    with open(os.path.join(HERE, "exact_tiny.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("exact_tiny.json", len(out))


class _CoinStream:
    """Stands in for the numpy Generator of SimState: `integers(2)` returns
    the next supplied coin (one per random collapse, tableau_sim.py:177)."""

    def __init__(self, coins):
        self.coins = coins
        self.k = 0

    def integers(self, n, *a, **kw):
        assert n == 2, n
        c = int(self.coins[self.k])
        self.k += 1
        return c


def refsample_cases():
    cases = [("d3", gen.surface_code_memory(3, 3, 1e-3)),
             ("d5", gen.surface_code_memory(5, 5, 5e-3)),
             ("d9", gen.surface_code_memory(9, 4, 1e-3)),
             ("c1", gen.random_clifford(64, 200, 0.01, 0)),
             ("c1b", gen.random_clifford(24, 60, 0.0, 3))]
    cases += [(name, text) for name, text, _, _, _ in mixed_cases()]
    return cases


def gen_refsample():
    _, rcircuit, _, _, _, _, tableau_sim = _ref()
    for i, (name, text) in enumerate(refsample_cases()):
        rc = rcircuit.parse(mc.to_reference_dialect(text))
        n_coll = sum(len(ins.targets) for ins in rcircuit.iter_flat(rc)
                     if ins.gate.name in ("M", "R", "MR"))
        coins = np.random.default_rng(300 + i).integers(0, 2, size=max(n_coll, 1), dtype=np.uint8)
        st = tableau_sim.SimState(rc.num_qubits, rng=_CoinStream(coins))
        bits = st.run(rc, skip_noise=True)
        np.savez_compressed(os.path.join(HERE, f"refsample_{name}.npz"), text=np.array(text),
                            coins=coins, used=st.rng.k, bits=np.array(bits, dtype=np.uint8),
                            determined=np.array(st.determined_record, dtype=np.uint8))
        print(f"refsample {name}: M={len(bits)} collapses={st.rng.k}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) == 3 and sys.argv[1] == "_statjob":
        import pickle
        with open(sys.argv[2], "rb") as f:
            job = pickle.load(f)
        with open(sys.argv[2] + ".out", "wb") as f:
            pickle.dump(_stat_worker(job), f)
        sys.exit(0)
    which = set(sys.argv[1:]) or {"plans", "inject", "noiseless", "stats", "exact", "refsample"}
    if "refsample" in which:
        gen_refsample()
    if "plans" in which:
        gen_frame_plans()
    if "exact" in which:
        gen_exact()
    if "inject" in which:
        gen_inject()
    if "noiseless" in which:
        gen_noiseless()
    if "stats" in which:
        gen_stats(min(8, os.cpu_count() or 1))
    for w in which:
        if w.startswith("stats_"):
            gen_stats(min(8, os.cpu_count() or 1), only={w[6:]})
