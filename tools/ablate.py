"""Kernel-time ablations for the frame kernel (profiling only; results of
skipped variants are wrong by construction).

    python tools/ablate.py [--config 2] [--shots N]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PFS_PROFILE", "1")  # profiling build of libpfs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--shots", type=int, default=1 << 18)
    ap.add_argument("--variants", default="")
    ap.add_argument("--groups", type=int, default=0)
    ap.add_argument("--words", type=int, default=0)
    ap.add_argument("--presample", type=int, default=0)
    a = ap.parse_args()
    import torch

    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    text = gen.config_circuit(a.config)
    variants = [
        ("base", {}),
        ("no_noise", {"debug_skip": 2}),
        ("no_coins", {"debug_skip": 4}),
        ("no_dets", {"debug_skip": 8}),
        ("no_gates", {"debug_skip": 16}),
        ("no_collapse", {"debug_skip": 32}),
        ("nothing", {"debug_skip": 2 | 8 | 16 | 32}),
        ("nn_no_gates", {"debug_skip": 2 | 16}),
        ("nn_no_collapse", {"debug_skip": 2 | 32}),
        ("nn_no_dets", {"debug_skip": 2 | 8}),
        ("gates_only", {"debug_skip": 2 | 8 | 32}),
        ("G1_W16", {"words_per_tile": 16, "groups": 1}),
        ("G4_W4", {"words_per_tile": 4, "groups": 4}),
        ("fused05", {"fused_target_hits": 0.5}),
        ("fused2", {"fused_target_hits": 2.0}),
    ]
    if a.variants:
        keep = set(a.variants.split(","))
        variants = [v for v in variants if v[0] in keep]
    res = {}
    for name, kw in variants:
        kw = dict(kw)
        if a.groups and "groups" not in kw:
            kw["groups"] = a.groups
        if a.words and "words_per_tile" not in kw:
            kw["words_per_tile"] = a.words
        kw.setdefault("presample_noise", a.presample)
        ds = compile_detector_sampler(text, timing=True, **kw)
        nb = (ds.num_columns + 7) // 8
        out = torch.empty((ds.num_columns, (a.shots + 31) // 32 + 64), dtype=torch.int32,
                          device="cuda")
        ts = []
        for i in range(4):
            ds.sample_rows(a.shots, seed=i, out=out[:, :(a.shots + 31) // 32])
            torch.cuda.synchronize()
            lt = ds.native.last_timing()
            ts.append((lt[0], lt[5]))
        best = min(ts[1:])
        res[name] = {"frame_ms": best[0], "noise_ms": best[1], "W": ds.info["words_per_tile"],
                     "threads": ds.info["threads"], "ring_smem": ds.info["ring_in_smem"]}
        print(name, json.dumps(res[name]), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
