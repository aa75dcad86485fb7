"""Summarise an ncu --page source --print-source sass CSV: stall totals and the
hottest SASS instructions (with a window of context)."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    col = {h: i for i, h in enumerate(hdr)}
    S = col["Warp Stall Sampling (All Samples)"]
    I = col["Instructions Executed"]
    tot_s = sum(float(r[S] or 0) for r in data)
    tot_i = sum(float(r[I] or 0) for r in data)
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    print("stall breakdown:")
    for h in sorted(stalls, key=lambda h: -sum(float(r[col[h]] or 0) for r in data)):
        v = sum(float(r[col[h]] or 0) for r in data)
        if v / tot_s > 0.01:
            print(f"  {h:28s} {100 * v / tot_s:5.1f}%")
    print(f"total samples {tot_s:.0f}, warp instrs {tot_i:.0f}")
    order = sorted(range(len(data)), key=lambda i: -float(data[i][S] or 0))[:top]
    for i in sorted(order):
        r = data[i]
        main_stall = max(stalls, key=lambda h: float(r[col[h]] or 0))
        print(f"{i:5d} {100 * float(r[S]) / tot_s:5.1f}% inst={float(r[I] or 0) / tot_i * 100:5.2f}% "
              f"{main_stall[6:]:14s} {r[1].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
