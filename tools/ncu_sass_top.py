"""Opcode mix and hottest SASS regions of an `ncu --page source --csv --print-source sass` dump.
    python tools/ncu_sass_top.py dump.csv [N]"""
import csv, sys, re
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = {h: i for i, h in enumerate(rows[1])}
ops = Counter(); tot = 0; thr = 0
recs = []
for r in rows[2:]:
    if len(r) < 8: continue
    src = r[hdr["Source"]].strip()
    try:
        n = float(r[hdr["Instructions Executed"]]); t = float(r[hdr["Thread Instructions Executed"]])
        st = float(r[hdr["Warp Stall Sampling (All Samples)"]])
    except ValueError:
        continue
    m = re.match(r"(@!?U?P\d+\s+)?([A-Z0-9_.]+)", src)
    op = m.group(2).split(".")[0] if m else "?"
    ops[op] += n; tot += n; thr += t
    recs.append((n, t, st, src))
print(f"warp instr {tot:.0f}  avg active lanes {thr / max(tot, 1):.1f}")
for k, v in ops.most_common(28):
    print(f"  {k:10s} {100 * v / tot:5.1f}%  {v / 1e6:8.2f}M")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if N:
    print("--- top stall instructions")
    stt = sum(r[2] for r in recs)
    for i, r in sorted(enumerate(recs), key=lambda x: -x[1][2])[:N]:
        print(f"  #{i:5d} stall {100 * r[2] / stt:5.2f}% inst {r[0] / 1e6:6.2f}M lanes {r[1] / max(r[0], 1):4.1f}  {r[3][:90]}")
