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
    a = ap.parse_args()
    import torch

    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    text = gen.config_circuit(a.config)
    variants = [
        ("base", {}),
        ("no_noise_apply", {"debug_skip": 1}),
        ("no_noise", {"debug_skip": 3}),
        ("no_coins", {"debug_skip": 4}),
        ("no_dets", {"debug_skip": 8}),
        ("no_gates", {"debug_skip": 16}),
        ("no_collapse", {"debug_skip": 32}),
        ("only_barriers", {"debug_skip": 63}),
        ("W16_global", {"words_per_tile": 16, "ring_in_smem": 0}),
        ("W8_global", {"words_per_tile": 8, "ring_in_smem": 0}),
        ("G1_W16", {"words_per_tile": 16, "ring_in_smem": 0, "groups": 1}),
        ("G2_W8", {"words_per_tile": 8, "ring_in_smem": 0, "groups": 2}),
        ("G2_W4", {"words_per_tile": 4, "ring_in_smem": 0, "groups": 2}),
        ("G2_W8_512", {"words_per_tile": 8, "ring_in_smem": 0, "groups": 2, "threads": 512}),
        ("G1_W8_rs", {"words_per_tile": 8, "ring_in_smem": 1, "groups": 1}),
        ("G2_W4_rs", {"words_per_tile": 4, "ring_in_smem": 1, "groups": 2}),
        ("G1_W16_640", {"words_per_tile": 16, "ring_in_smem": 0, "groups": 1, "threads": 640}),
        ("W8_512thr", {"threads": 512}),
        ("W4_smem", {"words_per_tile": 4, "ring_in_smem": 1}),
        ("hits2", {"noise_target_hits": 2.0}),
        ("hits05", {"noise_target_hits": 0.5}),
        ("W16_prod128", {"words_per_tile": 16, "ring_in_smem": 0, "producer_threads": 128}),
        ("W16_prod384", {"words_per_tile": 16, "ring_in_smem": 0, "producer_threads": 384}),
        ("W16_hits4", {"words_per_tile": 16, "ring_in_smem": 0, "noise_target_hits": 4.0}),
        ("W16_no_noise", {"words_per_tile": 16, "ring_in_smem": 0, "debug_skip": 3}),
        ("W16_no_gates", {"words_per_tile": 16, "ring_in_smem": 0, "debug_skip": 16}),
        ("W16_no_dets", {"words_per_tile": 16, "ring_in_smem": 0, "debug_skip": 8}),
        ("nn_no_gates", {"debug_skip": 3 | 16}),
        ("nn_no_dets", {"debug_skip": 3 | 8}),
        ("nn_no_collapse", {"debug_skip": 3 | 32}),
        ("nn_no_coins", {"debug_skip": 3 | 4}),
        ("producers_only", {"debug_skip": 1 | 4 | 8 | 16 | 32}),
        ("producers_only_p512", {"debug_skip": 1 | 4 | 8 | 16 | 32, "producer_threads": 512}),
        ("prod128", {"producer_threads": 128}),
        ("prod384", {"producer_threads": 384}),
        ("thr512_prod128", {"threads": 512, "producer_threads": 128}),
        ("no_stage", {"debug_skip": 1024}),
        ("no_stage_no_noise", {"debug_skip": 1024 | 3}),
        ("no_gates_collapse_dets", {"debug_skip": 8 | 16 | 32}),
        ("noise_only", {"debug_skip": 4 | 8 | 16 | 32}),
        ("dets_only", {"debug_skip": 1 | 2 | 4 | 16 | 32}),
        ("gates_only", {"debug_skip": 1 | 2 | 4 | 8 | 32}),
        ("collapse_only", {"debug_skip": 1 | 2 | 8 | 16}),
        ("nothing", {"debug_skip": 1 | 2 | 4 | 8 | 16 | 32}),
        ("nothing_no_stage", {"debug_skip": 1 | 2 | 4 | 8 | 16 | 32 | 1024}),
        ("nothing_G1", {"debug_skip": 1 | 2 | 4 | 8 | 16 | 32, "groups": 1}),
        ("nothing_256", {"debug_skip": 1 | 2 | 4 | 8 | 16 | 32, "threads": 256}),
        ("gates_only_no_stage", {"debug_skip": 1 | 2 | 4 | 8 | 32 | 1024}),
    ]
    if a.variants:
        keep = set(a.variants.split(","))
        variants = [v for v in variants if v[0] in keep]
    res = {}
    for name, kw in variants:
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
