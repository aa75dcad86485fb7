"""One sampling call for ncu / compute-sanitizer captures.

    python tools/profile_run.py [--config 2] [--shots N] [--words W] [--ring R] [--mode b8|rows|counts]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--shots", type=int, default=1 << 16)
    ap.add_argument("--words", type=int, default=0)
    ap.add_argument("--ring", type=int, default=-1)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--mode", default="b8")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--debug-skip", type=int, default=0)
    ap.add_argument("--groups", type=int, default=0)
    ap.add_argument("--kernel", type=int, default=0)
    a = ap.parse_args()
    import torch

    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    ds = compile_detector_sampler(gen.config_circuit(a.config), words_per_tile=a.words,
                                  ring_in_smem=a.ring, threads=a.threads,
                                  debug_skip=a.debug_skip, groups=a.groups, kernel=a.kernel)
    nb = (ds.num_columns + 7) // 8
    pitch = (nb + 31) // 32 * 32
    if a.mode == "b8":
        out = torch.empty((a.shots, pitch), dtype=torch.uint8, device="cuda")
        for i in range(a.reps):
            ds.sample(a.shots, seed=i, out=out[:, :nb])
    elif a.mode == "rows":
        out = torch.empty((ds.num_columns, (a.shots + 31) // 32), dtype=torch.int32, device="cuda")
        for i in range(a.reps):
            ds.sample_rows(a.shots, seed=i, out=out)
    else:
        out = torch.zeros(ds.num_columns, dtype=torch.int64, device="cuda")
        for i in range(a.reps):
            ds.sample_counts(a.shots, seed=i, out=out)
    torch.cuda.synchronize()
    print("ok", ds.info)


if __name__ == "__main__":
    main()
