"""Group an ncu SASS source-page CSV into basic blocks (runs of equal
execution count) and list the blocks by executed warp instructions."""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path, errors="replace")))
    hdr = rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    I, S = col["Instructions Executed"], col["Warp Stall Sampling (All Samples)"]
    blocks, cur = [], None
    for k, r in enumerate(data):
        n = float(r[I] or 0)
        if cur is None or n != cur["n"]:
            cur = {"start": k, "n": n, "len": 0, "ops": [], "stall": 0.0}
            blocks.append(cur)
        cur["len"] += 1
        cur["stall"] += float(r[S] or 0)
        cur["ops"].append(r[col["Source"]].split()[0] if r[col["Source"]].split() else "")
    tot_i = sum(b["n"] * b["len"] for b in blocks)
    tot_s = sum(b["stall"] for b in blocks)
    print(f"total warp instrs {tot_i:.0f}, stall samples {tot_s:.0f}")
    for b in sorted(blocks, key=lambda b: -b["n"] * b["len"])[:top]:
        ops = " ".join(o for o in b["ops"][:14])
        print(f"sass#{b['start']:5d} len {b['len']:4d} x{b['n']:10.0f} = {100 * b['n'] * b['len'] / tot_i:5.1f}% instr,"
              f" {100 * b['stall'] / tot_s:5.1f}% stall | {ops}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
