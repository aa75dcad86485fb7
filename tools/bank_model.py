"""Host-side model of the gate passes' shared-memory bank conflicts (no GPU).

    python tools/bank_model.py [--config 2] [--words 8] [--groups 2]
For every gate op's per-warp operand block (pfs_program_dump) it counts, per quarter-warp
phase of a pass (128 B / row bytes applications), the conflict degree of each operand's
row accesses (rows in the same bank class = row mod classes) and reports wavefronts vs the
conflict-free count, per rule."""
import argparse, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--words", type=int, default=0)
    ap.add_argument("--groups", type=int, default=0)
    a = ap.parse_args()
    from paper_2103_02202_b200 import _native as N, generators as gen
    from paper_2103_02202_b200.program import flatten
    f = flatten(gen.config_circuit(a.config))
    p = N.NativeProgram(f, words_per_tile=a.words, groups=a.groups)
    info = p.info
    W = info["words_per_tile"]
    V = 4 if W >= 4 else W
    C = W // V
    PI = 32 // C
    classes = 1 if W >= 32 else 128 // (W * 4)
    q = max(1, 8 // C) if V == 4 else 32 // max(1, classes // 1)  # applications per quarter-warp phase (128-bit accesses)
    q = classes  # applications one wavefront can serve
    wpg = info["threads"] // int(info["groups"]) // 32
    ops = p.dump(0).reshape(-1, 8)
    sops = p.dump(4).reshape(-1, 12)
    arena = p.dump(5)
    n = f.num_qubits
    tot = {}
    for op, so in zip(ops, sops):
        if (int(op[0]) & 0xFF) != 0:
            continue
        code = (int(op[0]) >> 8) & 0xFF
        ar = 2 if code >= 4 else 1
        K = int(so[3])
        stride = max(K, 4) * PI
        blk = arena[int(so[2]): int(so[2]) + wpg * stride].reshape(wpg, stride)
        wf = ideal = 0
        for w in range(wpg):
            for k in range(K):
                words = blk[w, k * PI:(k + 1) * PI]
                for g0 in range(0, PI, q):
                    grp = words[g0:g0 + q]
                    for s in range(ar):
                        rows = (grp >> (16 * s)) & 0xFFFF
                        deg = np.bincount(rows % classes, minlength=classes).max()
                        wf += deg
                        ideal += 1
        t = tot.setdefault(code, [0, 0, 0])
        t[0] += 1; t[1] += wf; t[2] += ideal
    print(info["words_per_tile"], "words/tile,", classes, "bank classes,", wpg, "warps per group")
    for code, (nops, wf, ideal) in sorted(tot.items()):
        print(f"rule {code}: {nops} ops, row-access wavefronts {wf} vs conflict-free {ideal}: x{wf / ideal:.3f}")


if __name__ == "__main__":
    main()
