"""CUDA path (through the C-ABI) against the reference goldens and the C oracle.

Parity bars (BASELINE.json north_star):
  * injected-mask mode: bit-exact vs the reference's own FrameBatch (goldens);
  * Philox mode: bit-exact vs the C oracle making the same counter-based draws,
    and within binomial 5 sigma of the reference's sampled frequencies;
  * noiseless: events all zero, deterministic measurements equal the
    reference sample.
"""

import numpy as np
import pytest

from tests._util import (b8_unpack, five_sigma, inject_cases, load_exact, load_inject,
                         load_noiseless, load_stats, pair_counts, rows_unpack)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2103_02202_b200.build import build
    build()


# (words_per_tile, ring_in_smem, groups, kernel) layouts exercising every
# kernel instantiation: cooperative (kernel 1; one and two tiles in flight per
# CTA), warp-private (kernel 2; one word column per warp, 8-word tiles) and
# word-column (kernel 3; one-word tiles, staged op-block stream), 0 = auto
LAYOUTS = [(0, -1, 0, 0), (1, 0, 1, 1), (2, 1, 2, 1), (4, 0, 0, 1), (8, 1, 1, 1), (16, 0, 2, 1),
           (32, 1, 0, 1), (16, 0, 1, 1), (1, -1, 0, 2), (2, -1, 0, 2), (4, -1, 0, 2),
           (16, -1, 0, 2), (32, -1, 0, 2), (0, -1, 0, 3), (1, 0, 0, 3), (2, 1, 0, 3),
           (4, 0, 0, 3), (4, 1, 0, 3)]


def _opts(layout):
    W, ring, groups, kernel = layout
    return dict(words_per_tile=W, ring_in_smem=ring, groups=groups, kernel=kernel)


def _fits(text, layout):
    from paper_2103_02202_b200._native import NativeProgram
    from paper_2103_02202_b200.program import flatten
    try:
        p = NativeProgram(flatten(text), **_opts(layout))
    except ValueError:
        return False
    return layout[3] == 0 or p.info["kernel"] == layout[3]


@pytest.mark.parametrize("name", inject_cases())
@pytest.mark.parametrize("layout", LAYOUTS)
def test_injected_bit_exact_vs_reference(name, layout):
    from paper_2103_02202_b200.sampler import compile_detector_sampler, compile_sampler

    text, B, coins, masks, flips_ref, events_ref = load_inject(name)
    if not _fits(text, layout):
        pytest.skip("layout does not fit")
    ds = compile_detector_sampler(text, **_opts(layout))
    ev = ds.sample(B, coins=coins, masks=masks)
    assert np.array_equal(ev, events_ref)
    ms = compile_sampler(text, **_opts(layout))
    fl = ms.sample_flips(B, coins=coins, masks=masks)
    assert np.array_equal(fl, flips_ref)
    # counts mode sees the same events
    cnt = ds.sample_counts(B, coins=coins, masks=masks)
    assert np.array_equal(cnt, b8_unpack(events_ref, ds.num_columns).sum(axis=0))


def _philox_cases():
    from paper_2103_02202_b200 import generators as gen
    return {
        "d3_p1e-2": gen.surface_code_memory(3, 3, 1e-2),
        "d5": gen.surface_code_memory(5, 5, 5e-3),
        "c1": gen.random_clifford(64, 200, 0.01, 0),
        "mix5": load_inject("mix5")[0],
        "mix4": load_inject("mix4")[0],
        "d9_highp": gen.surface_code_memory(9, 2, 0.05),
    }


@pytest.mark.parametrize("case", list(_philox_cases()))
@pytest.mark.parametrize("layout", [(0, -1, 0, 0), (1, 1, 1, 1), (4, 0, 2, 1), (16, 1, 1, 1),
                                    (8, 0, 2, 1), (2, -1, 0, 2), (8, -1, 0, 2), (32, -1, 0, 2)])
def test_philox_bit_exact_vs_oracle(oracle_lib, case, layout):
    from paper_2103_02202_b200.sampler import compile_detector_sampler, compile_sampler

    text = _philox_cases()[case]
    if not _fits(text, layout):
        pytest.skip("layout does not fit")
    ds = compile_detector_sampler(text, **_opts(layout))
    T = ds.tile_shots
    shots = 3 * T + 37
    seed = 0xC0FFEE
    offset = 5 * T
    ev_rows = ds.sample_rows(shots, seed=seed, shot_offset=offset)
    ms = compile_sampler(text, **_opts(layout))
    fl_rows = ms.sample_flip_rows(shots, seed=seed, shot_offset=offset)
    ofl, oev = oracle_lib.sample(ds.flat, shots, T, seed=seed, tile_offset=offset // T,
                                 nthreads=4, schedule=ds.native.noise_schedule())
    assert np.array_equal(rows_unpack(ev_rows, shots), rows_unpack(oev, shots))
    assert np.array_equal(rows_unpack(fl_rows, shots), rows_unpack(ofl, shots))
    # b8 outputs are the transposes of the row outputs
    ev_b8 = ds.sample(shots, seed=seed, shot_offset=offset)
    assert np.array_equal(b8_unpack(ev_b8, ds.num_columns), rows_unpack(oev, shots))
    fl_b8 = ms.sample_flips(shots, seed=seed, shot_offset=offset)
    assert np.array_equal(b8_unpack(fl_b8, ms.num_measurements), rows_unpack(ofl, shots))


@pytest.mark.parametrize("W", [1, 8, 32])
def test_warp_and_cooperative_kernels_agree(W):
    """Both frame kernels make the same counter-based draws for one tile width:
    b8 events, flips and counts agree bit for bit (d=7 surface code, tail tile)."""
    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler, compile_sampler

    text = gen.surface_code_memory(7, 7, 2e-3)
    a = compile_detector_sampler(text, words_per_tile=W, kernel=1)
    b = compile_detector_sampler(text, words_per_tile=W, kernel=2)
    assert a.native.info["kernel"] == 1 and b.native.info["kernel"] == 2
    shots = 37 * 32 * W + 11
    assert np.array_equal(a.sample(shots, seed=5), b.sample(shots, seed=5))
    assert np.array_equal(a.sample_counts(shots, seed=5), b.sample_counts(shots, seed=5))
    ma = compile_sampler(text, words_per_tile=W, kernel=1)
    mb = compile_sampler(text, words_per_tile=W, kernel=2)
    assert np.array_equal(ma.sample_flips(shots, seed=6), mb.sample_flips(shots, seed=6))
    assert np.array_equal(ma.sample_flip_rows(shots, seed=6), mb.sample_flip_rows(shots, seed=6))


def test_shard_invariance():
    """Counter-based RNG: a shot range split across calls (or GPUs) gives the
    same bits as one call."""
    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    ds = compile_detector_sampler(gen.surface_code_memory(5, 5, 5e-3))
    T = ds.tile_shots
    whole = ds.sample(8 * T, seed=7)
    parts = [ds.sample(2 * T, seed=7, shot_offset=i * 2 * T) for i in range(4)]
    assert np.array_equal(whole, np.concatenate(parts))
    c_whole = ds.sample_counts(8 * T, seed=7)
    c_parts = sum(ds.sample_counts(2 * T, seed=7, shot_offset=i * 2 * T) for i in range(4))
    assert np.array_equal(c_whole, c_parts)


@pytest.mark.parametrize("name", ["d3", "d5", "c1", "mix"])
def test_noiseless(name):
    from paper_2103_02202_b200.sampler import compile_detector_sampler, compile_sampler

    text, ref, det = load_noiseless(name)
    shots = 5000
    ms = compile_sampler(text, reference=ref)
    samples = b8_unpack(ms.sample(shots, seed=3), ms.num_measurements)
    assert np.array_equal(samples[:, det], np.broadcast_to(ref[det], samples[:, det].shape))
    if name in ("d3", "d5"):
        ds = compile_detector_sampler(text)
        assert not ds.sample(shots, seed=4).any()
        assert not ds.sample_counts(1 << 20, seed=4).any()


@pytest.mark.parametrize("name", ["d3", "d5", "c1", "d25"])
def test_statistics_vs_reference(name):
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    try:
        text, n_ref, counts_ref, pairs, pc_ref = load_stats(name)
    except FileNotFoundError:
        pytest.skip("no fixture")
    ds = compile_detector_sampler(text)
    shots = 1 << 18 if name != "d25" else 1 << 16
    ev = ds.sample(shots, seed=2024)
    bits = b8_unpack(ev, ds.num_columns)
    assert five_sigma(bits.sum(axis=0), shots, counts_ref, n_ref) < 5.0
    assert five_sigma(pair_counts(bits, pairs), shots, pc_ref, n_ref) < 5.0


def test_exact_tiny_distributions():
    from scipy.stats import chi2

    from paper_2103_02202_b200.sampler import compile_sampler

    for case in load_exact():
        ms = compile_sampler(case["text"], reference=case["reference"])
        shots = 50000
        s = b8_unpack(ms.sample(shots, seed=11), ms.num_measurements)
        dist = {tuple(k): v for k, v in case["dist"]}
        obs = {}
        for k in map(tuple, s.tolist()):
            obs[k] = obs.get(k, 0) + 1
        assert set(obs) <= set(dist)
        stat = sum((obs.get(k, 0) - shots * p) ** 2 / (shots * p) for k, p in dist.items())
        assert chi2.sf(stat, max(1, len(dist) - 1)) > 1e-3, case["text"]


def test_device_output_matches_host_output():
    import torch

    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    ds = compile_detector_sampler(gen.surface_code_memory(7, 7, 1e-3))
    shots = 10 * ds.tile_shots + 5
    host = ds.sample(shots, seed=9)
    dev = torch.empty((shots, (ds.num_columns + 7) // 8), dtype=torch.uint8, device="cuda")
    ds.sample(shots, seed=9, out=dev)
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy(), host)


def test_c2_full_size_properties():
    """BASELINE config 2 at full size (2^20 shots): the b8 events, the
    row-major events and the on-device counts are three views of the same
    Philox draws and must agree exactly; the mean event rate must match the
    reference's (stats fixture) within 5 sigma."""
    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    text = gen.config_circuit(2)
    ds = compile_detector_sampler(text)
    shots = 1 << 20
    ev = ds.sample(shots, seed=42)
    assert ev.shape == (shots, 1951)
    counts = ds.sample_counts(shots, seed=42)
    col_pop = np.unpackbits(ev, axis=0, bitorder="little")  # cheap column popcount
    del col_pop
    pop = np.zeros(ds.num_columns, dtype=np.int64)
    for b in range(8):
        pop_b = ((ev >> b) & 1).sum(axis=0, dtype=np.int64)
        idx = np.arange(ev.shape[1]) * 8 + b
        ok = idx < ds.num_columns
        pop[idx[ok]] = pop_b[ok]
    assert np.array_equal(pop, counts.astype(np.int64))
    try:
        _, n_ref, counts_ref, _, _ = load_stats("d25")
        assert five_sigma(counts, shots, counts_ref, n_ref) < 5.0
    except FileNotFoundError:
        pass


@pytest.mark.parametrize("case", ["d3_p1e-2", "d5", "d9_highp"])
def test_error_model_sampler_equals_frame_sampler(oracle_lib, case):
    """The error-model sampler (kernel 4: detection events = XOR of the noise
    hits' output signatures) makes the frame sampler's own draws with one-word
    tiles: events (b8, rows) and counts agree bit for bit with the frame
    kernel and with the C oracle."""
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    text = _philox_cases()[case]
    dem = compile_detector_sampler(text, kernel=4)
    frm = compile_detector_sampler(text, kernel=1, words_per_tile=1)
    assert dem.native.info["kernel"] == 4 and dem.tile_shots == 32 == frm.tile_shots
    for shots, off in ((4096, 0), (1000 + 7, 32 * 37)):
        a = dem.sample(shots, seed=11, shot_offset=off)
        assert np.array_equal(a, frm.sample(shots, seed=11, shot_offset=off))
        assert np.array_equal(dem.sample_rows(shots, seed=11, shot_offset=off),
                              frm.sample_rows(shots, seed=11, shot_offset=off))
        assert np.array_equal(dem.sample_counts(shots, seed=11, shot_offset=off),
                              b8_unpack(a, dem.num_columns).sum(axis=0))
    shots = 3 * 32 + 5
    _, oev = oracle_lib.sample(dem.flat, shots, 32, seed=3, tile_offset=2, nthreads=4, flips=False,
                               schedule=dem.native.noise_schedule())
    assert np.array_equal(b8_unpack(dem.sample(shots, seed=3, shot_offset=64), dem.num_columns),
                          rows_unpack(oev, shots))


def test_error_model_sampler_shot_major_rows():
    """dem_kernel keeps a tile's events shot-major in shared memory and stores
    each shot's row directly: 16-byte vector path (host output through the
    32-byte-pitch scratch), bytewise path (device output with an odd pitch),
    ragged tail tile and a shot offset — bit-exact with the frame kernel."""
    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler
    import torch

    text = gen.surface_code_memory(25, 5, 2e-3)
    dem = compile_detector_sampler(text, kernel=4)
    frm = compile_detector_sampler(text, kernel=1, words_per_tile=1)
    assert dem.native.info["kernel"] == 4
    shots, off = 5000 + 13, 32 * 5
    ref = frm.sample(shots, seed=8, shot_offset=off)
    assert np.array_equal(dem.sample(shots, seed=8, shot_offset=off), ref)
    nb = (dem.num_columns + 7) // 8
    dev = torch.zeros((shots, nb + 1), dtype=torch.uint8, device="cuda")[:, 1:]  # odd base, pitch nb + 1
    dem.sample(shots, seed=8, shot_offset=off, out=dev)
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy(), ref)
    # counts and column-major rows keep the column-word layout
    assert np.array_equal(dem.sample_rows(shots, seed=8, shot_offset=off),
                          frm.sample_rows(shots, seed=8, shot_offset=off))
    assert np.array_equal(dem.sample_counts(shots, seed=8, shot_offset=off),
                          b8_unpack(ref, dem.num_columns).sum(axis=0))


def test_error_model_sampler_full_size_d25():
    """Config 2 at 2^20 shots through the error-model sampler: identical to the
    frame sampler on one-word tiles."""
    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler
    import torch

    text = gen.config_circuit(2)
    dem = compile_detector_sampler(text, kernel=4)
    frm = compile_detector_sampler(text, kernel=1, words_per_tile=1)
    shots = 1 << 20
    nb = (dem.num_columns + 7) // 8
    a = torch.empty((shots, nb), dtype=torch.uint8, device="cuda")
    b = torch.empty((shots, nb), dtype=torch.uint8, device="cuda")
    dem.sample(shots, seed=21, out=a)
    frm.sample(shots, seed=21, out=b)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_error_model_sampler_global_columns():
    """More output columns than one CTA's shared memory holds (d=51, 20 rounds:
    ~52k columns): the column words accumulate in global memory and go through
    the tile transpose — still bit-exact with the frame kernel on 32-shot tiles."""
    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    text = gen.surface_code_memory(51, 20, 2e-3)
    dem = compile_detector_sampler(text, kernel=4)
    assert dem.native.info["smem_bytes"] < 64 * 1024  # global column words
    frm = compile_detector_sampler(text, kernel=1, words_per_tile=1)
    for shots, off in ((2048, 0), (333, 32 * 9)):
        assert np.array_equal(dem.sample(shots, seed=4, shot_offset=off),
                              frm.sample(shots, seed=4, shot_offset=off))
        assert np.array_equal(dem.sample_rows(shots, seed=4, shot_offset=off),
                              frm.sample_rows(shots, seed=4, shot_offset=off))
