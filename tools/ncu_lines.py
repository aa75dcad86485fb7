"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump by CUDA
source line: warp instructions, stall samples, shared wavefronts (top N)."""
import csv
import sys


def main(path, top=45):
    rows = list(csv.reader(open(path)))
    out = []
    fname = ""
    hdr = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) > 10 and r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or len(r) < 10 or not r[0].isdigit():
            continue
        try:
            ins = float(r[hdr["Instructions Executed"]] or 0)
            smp = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
            wf = float(r[hdr["L1 Wavefronts Shared"]] or 0)
            wfi = float(r[hdr["L1 Wavefronts Shared Ideal"]] or 0)
        except ValueError:
            continue
        if ins or smp:
            out.append((fname, int(r[0]), r[1].strip()[:80], ins, smp, wf, wfi))
    ti = sum(o[3] for o in out)
    ts = sum(o[4] for o in out)
    print(f"total warp instrs {ti:.0f} samples {ts:.0f} wavefronts {sum(o[5] for o in out):.0f} "
          f"ideal {sum(o[6] for o in out):.0f}")
    for o in sorted(out, key=lambda o: -o[3])[:top]:
        print(f"{o[0][:14]:14s}:{o[1]:5d} inst {100 * o[3] / ti:5.2f}% stall {100 * o[4] / ts:5.2f}% "
              f"wf {o[5] / 1e6:6.2f}M/{o[6] / 1e6:6.2f}M  {o[2]}")
    print("--- by stall samples")
    for o in sorted(out, key=lambda o: -o[4])[:25]:
        print(f"{o[0][:14]:14s}:{o[1]:5d} inst {100 * o[3] / ti:5.2f}% stall {100 * o[4] / ts:5.2f}%  {o[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 45)
