"""Small sampling calls for compute-sanitizer (racecheck / synccheck / memcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Runs, through the public sampler, on tiny shot counts (the sanitizer slows
kernels ~100x): config 0 (d=3 surface code) and the mixed golden circuits with
duplicate targets / `CX 0 1 1 2` conflicts (tests/golden/inject_mix*.npz), each
in injected-mask mode (bit-exact vs the reference golden) and in Philox mode,
for detection events, measurement flips and on-device counts, on several tile
layouts.  Exits non-zero on any mismatch.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np

    from _util import load_inject
    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler, compile_sampler

    names = ["c0_d3", "mix0", "mix3", "mix7"]
    layouts = [dict(), dict(words_per_tile=1), dict(words_per_tile=2, ring_in_smem=0), dict(words_per_tile=8, groups=2)]
    n = 0
    for name in names:
        text, B, coins, masks, flips_b8, events_b8 = load_inject(name)
        for lay in layouts:
            ds = compile_detector_sampler(text, device=0, **lay)
            ev = ds.sample(B, coins=coins, masks=masks)
            assert np.array_equal(ev, events_b8), ("injected events", name, lay)
            T = ds.tile_shots
            ds.sample(3 * T + 5, seed=7)          # Philox mode, ragged tail
            ds.sample_counts(2 * T, seed=9)
            n += 3
        ms = compile_sampler(text, device=0)   # record flavour (measurement flips)
        fl = ms.sample_flips(B, coins=coins, masks=masks)
        assert np.array_equal(fl, flips_b8), ("injected flips", name)
        ms.sample_flips(2 * ms.tile_shots + 3, seed=11)
        n += 2
    # config 1 (random Clifford, standalone noise ops, MR) in Philox mode
    ds = compile_detector_sampler(gen.config_circuit(1), device=0)
    ds.sample(2 * ds.tile_shots, seed=3)
    n += 1
    print("sanitize_run ok:", n, "calls")


if __name__ == "__main__":
    main()
