"""Per-op time of the frame kernel from clock64 traces (profiling only).

    python tools/op_trace.py [--config 2] [--shots N]
Prints the cycle share per op kind (and the costliest ops)."""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PFS_PROFILE", "1")  # profiling build of libpfs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--shots", type=int, default=1 << 16)
    ap.add_argument("--groups", type=int, default=0)
    ap.add_argument("--words", type=int, default=0)
    ap.add_argument("--debug", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--kernel", type=int, default=0)
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    ds = compile_detector_sampler(gen.config_circuit(a.config), debug_skip=64 | a.debug, groups=a.groups,
                                  words_per_tile=a.words, kernel=a.kernel, threads=a.threads)
    out = torch.empty((ds.num_columns, (a.shots + 31) // 32), dtype=torch.int32, device="cuda")
    for i in range(3):
        ds.sample_rows(a.shots, seed=i, out=out)
    torch.cuda.synchronize()
    clk9 = ds.native.op_clock()
    clk = clk9[0]
    ends = clk9[1:9]  # per-warp (warps 0..7) end of each op's work
    top_t, gate_t, hdr_t = clk9[9], clk9[10], clk9[11]  # warp 0: op top, gate rows done, header done
    ops = ds.native.ops()
    dt = np.diff(clk)
    work = ends[:, :-1] - clk[None, :-1]  # per warp: op start (barrier exit) -> own work done
    names = {0: "GATE", 1: "M", 2: "R", 3: "MR", 4: "NOISE", 5: "DET", 6: "OBS", 7: "SPILL"}
    agg = collections.defaultdict(lambda: [0, 0])
    for i, d in enumerate(dt):
        k = int(ops[i, 0] & 0xFF)
        key = names.get(k, str(k)) + ("/bar" if (ops[i + 1, 0] >> 16) & 1 else "")
        agg[key][0] += 1
        agg[key][1] += int(d)
    tot = int(dt.sum())
    print(ds.info)
    print(f"first tile: {tot} cycles over {len(dt)} ops")
    for k, (n, c) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {k:12s} n={n:4d} cycles={c:9d} ({100 * c / tot:5.1f}%)  avg={c / n:8.0f}")
    # per (kind, code) breakdown
    agg2 = collections.defaultdict(lambda: [0, 0, 0])
    for i, d in enumerate(dt):
        k = int(ops[i, 0] & 0xFF)
        key = (names.get(k, str(k)), int((ops[i, 0] >> 8) & 0xFF))
        agg2[key][0] += 1
        agg2[key][1] += int(d)
        agg2[key][2] += int(ops[i, 1])
    wk = collections.defaultdict(list)
    for i in range(len(dt)):
        k = int(ops[i, 0] & 0xFF)
        wk[(names.get(k, str(k)), int((ops[i, 0] >> 8) & 0xFF))].append(work[:, i])
    for k, (n, c, cnt) in sorted(agg2.items(), key=lambda x: -x[1][1]):
        w = np.array(wk[k])
        print(f"  {k[0]:6s} code={k[1]} n={n:4d} avg_cycles={c / n:8.0f} avg_count={cnt / n:8.1f} "
              f"warp0_work={w[:, 0].mean():7.0f} warpmax_work={w.max(axis=1).mean():7.0f} "
              f"warpmin_work={w.min(axis=1).mean():7.0f}")
    # warp 0 phases: header (top -> at barrier), barrier wait (-> op start), gate rows, noise / rest
    print("  warp 0 phases per op kind: header | barrier wait | gate rows | rest (noise, collapses, detectors)")
    ph = collections.defaultdict(lambda: [0, 0, 0, 0, 0])
    for i in range(len(dt)):
        k = int(ops[i, 0] & 0xFF)
        key = (names.get(k, str(k)), int((ops[i, 0] >> 8) & 0xFF))
        p = ph[key]
        p[0] += 1
        p[1] += int(hdr_t[i] - top_t[i])
        p[2] += int(clk[i] - hdr_t[i])
        if gate_t[i] > 0:
            p[3] += int(gate_t[i] - clk[i])
            p[4] += int(ends[0, i] - gate_t[i])
        else:
            p[4] += int(ends[0, i] - clk[i])
    for k, p in sorted(ph.items()):
        n = p[0]
        print(f"  {k[0]:6s} code={k[1]} n={n:4d} header={p[1] / n:7.0f} barrier={p[2] / n:7.0f} gate={p[3] / n:7.0f} rest={p[4] / n:7.0f}")
    top = np.argsort(dt)[::-1][:5]
    for i in top:
        print(f"  op {i:4d} kind={names.get(int(ops[i, 0] & 0xFF))} code={(ops[i, 0] >> 8) & 0xFF} "
              f"count={ops[i, 1]} cycles={dt[i]}")


if __name__ == "__main__":
    main()
