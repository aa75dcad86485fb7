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
                         load_noiseless, load_stats, oracle_run, pair_counts, rows_unpack)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2103_02202_b200.build import build
    build()


# (words_per_tile, ring_in_smem, groups, kernel) layouts exercising every
# frame-kernel instantiation: W in {1..32} x ring in shared / global memory,
# one to four tiles in flight per CTA, 0 = auto
LAYOUTS = [(0, -1, 0, 0), (1, 0, 1, 1), (1, 1, 2, 1), (2, 1, 2, 1), (2, 0, 1, 1), (4, 0, 0, 1),
           (4, 1, 4, 1), (8, 1, 1, 1), (8, 0, 2, 1), (16, 0, 2, 1), (16, 1, 1, 1), (32, 1, 0, 1),
           (32, 0, 1, 1)]


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
                                    (8, 0, 2, 1), (2, 0, 4, 1), (32, 0, 1, 1)])
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
    ofl, oev = oracle_run(oracle_lib, ds, shots, seed, offset, nthreads=4)
    assert np.array_equal(rows_unpack(ev_rows, shots), rows_unpack(oev, shots))
    assert np.array_equal(rows_unpack(fl_rows, shots), rows_unpack(ofl, shots))
    # b8 outputs are the transposes of the row outputs
    ev_b8 = ds.sample(shots, seed=seed, shot_offset=offset)
    assert np.array_equal(b8_unpack(ev_b8, ds.num_columns), rows_unpack(oev, shots))
    fl_b8 = ms.sample_flips(shots, seed=seed, shot_offset=offset)
    assert np.array_equal(b8_unpack(fl_b8, ms.num_measurements), rows_unpack(ofl, shots))


def test_tile_index_above_2_32(oracle_lib):
    """Tiles past 2^32 (shot offsets ~1e12) fold the tile index's high bits into
    the Philox key: distinct streams, still bit-exact with the oracle."""
    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    ds = compile_detector_sampler(gen.surface_code_memory(5, 5, 5e-3))
    T = ds.tile_shots
    low = 7 * T
    high = ((1 << 32) + 7) * T
    a = ds.sample_rows(2 * T, seed=11, shot_offset=low)
    b = ds.sample_rows(2 * T, seed=11, shot_offset=high)
    assert not np.array_equal(a, b)
    _, oev = oracle_run(oracle_lib, ds, 2 * T, 11, high, nthreads=2, flips=False)
    assert np.array_equal(rows_unpack(b, 2 * T), rows_unpack(oev, 2 * T))


@pytest.mark.parametrize("d", [5, 9])
def test_event_and_record_programs_agree(d):
    """The detection-event program (records kept in x rows, shared ring,
    irrelevant coins skipped) and the measurement-record program make the same
    noise draws: detector_events of the sampled flips equals the events."""
    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.circuit import detector_and_observable_sets, parse
    from paper_2103_02202_b200.sampler import compile_detector_sampler, compile_sampler

    text = gen.surface_code_memory(d, d, 4e-3)
    c = parse(text)
    ds = compile_detector_sampler(c)
    ms = compile_sampler(c)
    shots = 11 * ds.tile_shots + 3
    ev = b8_unpack(ds.sample(shots, seed=5, shot_offset=ds.tile_shots), ds.num_columns)
    fl = b8_unpack(ms.sample_flips(shots, seed=5, shot_offset=ds.tile_shots), ms.num_measurements)
    expect = np.stack([np.bitwise_xor.reduce(fl[:, list(s)], axis=1) for s in detector_and_observable_sets(c)],
                      axis=1)
    assert np.array_equal(ev, expect)


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


def _row_counts(rows, shots, pairs):
    """Per-column and pairwise event counts from column-major uint32 rows."""
    words = (shots + 31) // 32
    r = np.ascontiguousarray(rows[:, :words])
    tail = shots - 32 * (words - 1)
    if tail < 32:
        r[:, -1] &= np.uint32((1 << tail) - 1)
    counts = np.bitwise_count(r).sum(axis=1, dtype=np.int64)
    pc = np.zeros(len(pairs), dtype=np.int64)
    for i in range(0, len(pairs), 512):
        pp = pairs[i:i + 512]
        pc[i:i + 512] = np.bitwise_count(r[pp[:, 0]] & r[pp[:, 1]]).sum(axis=1, dtype=np.int64)
    return counts, pc


@pytest.mark.parametrize("name", ["d3", "d5", "c1", "d25"])
def test_statistics_vs_reference(name):
    """5 sigma per detector and per sampled detector pair against event counts
    of the reference's own collect_flips + detector_events
    (tests/golden/stats_*.npz; d25 = BASELINE config 2 at 2^20 reference shots)."""
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    text, n_ref, counts_ref, pairs, pc_ref = load_stats(name)  # missing fixture = failure
    ds = compile_detector_sampler(text)
    shots = 1 << 20
    rows = ds.sample_rows(shots, seed=2024)
    counts, pc = _row_counts(rows, shots, pairs)
    assert five_sigma(counts, shots, counts_ref, n_ref) < 5.0
    assert five_sigma(pc, shots, pc_ref, n_ref) < 5.0


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
    Philox draws and must agree exactly; the per-detector event rates must
    match the reference's (stats fixture, 2^20 reference shots) within 5 sigma."""
    import torch

    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    text = gen.config_circuit(2)
    ds = compile_detector_sampler(text)
    shots = 1 << 20
    nb = (ds.num_columns + 7) // 8
    dev = torch.empty((shots, nb), dtype=torch.uint8, device="cuda")
    ds.sample(shots, seed=42, out=dev)
    counts = ds.sample_counts(shots, seed=42)
    rows = ds.sample_rows(shots, seed=42)
    # column popcounts of the b8 events, on the device
    pop = torch.zeros(nb * 8, dtype=torch.int64, device="cuda")
    for b in range(8):
        pop[b::8] = ((dev >> b) & 1).sum(dim=0, dtype=torch.int64)
    pop = pop[:ds.num_columns].cpu().numpy()
    assert np.array_equal(pop, counts.astype(np.int64))
    assert np.array_equal(np.bitwise_count(rows).sum(axis=1, dtype=np.int64), counts.astype(np.int64))
    # first and last shot rows: b8 vs rows
    host = dev[:64].cpu().numpy()
    assert np.array_equal(b8_unpack(host, ds.num_columns), rows_unpack(rows[:, :2], 64))
    _, n_ref, counts_ref, _, _ = load_stats("d25")
    assert five_sigma(counts, shots, counts_ref, n_ref) < 5.0


def test_c2_bench_layout_bit_exact_vs_oracle(oracle_lib):
    """Config 2 through the bench's own layout (W=8, two tiles per CTA, 640
    threads, sub-chunk pipeline of frame kernel and transposes, device b8
    output, nonzero offset) over more than two waves of tiles: the first,
    middle and last tiles are bit-exact with the oracle."""
    import torch

    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    ds = compile_detector_sampler(gen.config_circuit(2))
    info = ds.info
    assert info["words_per_tile"] == 8 and info["groups"] == 2 and info["threads"] == 640
    T = ds.tile_shots
    n_tiles = 2 * 148 * 2 + 9
    shots = n_tiles * T - 77
    off = 13 * T
    nb = (ds.num_columns + 7) // 8
    dev = torch.empty((shots, nb), dtype=torch.uint8, device="cuda")
    ds.sample(shots, seed=20260214, out=dev, shot_offset=off)
    torch.cuda.synchronize()
    for t0, nt in ((0, 4), (n_tiles // 2, 4), (n_tiles - 3, 3)):
        s0 = t0 * T
        ns = min(nt * T, shots - s0)
        _, oev = oracle_run(oracle_lib, ds, ns, 20260214, off + s0, nthreads=8, flips=False)
        got = dev[s0:s0 + ns].cpu().numpy()
        assert np.array_equal(b8_unpack(got, ds.num_columns), rows_unpack(oev, ns)), t0


@pytest.mark.parametrize("ring", [-1, 0])
def test_c4_d100_bit_exact_vs_oracle(oracle_lib, ring):
    """Config 4 (d=100, 100 rounds: 20k qubits, 1M records): one-word tiles,
    the record ring in shared memory (auto) or global memory — detection
    events bit-exact with the oracle on 4 tiles at a nonzero offset."""
    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    ds = compile_detector_sampler(gen.config_circuit(4), ring_in_smem=ring)
    assert ds.info["words_per_tile"] == 1
    if ring == -1:
        assert ds.info["ring_in_smem"] == 1
    T = ds.tile_shots
    shots, off = 4 * T - 5, 3 * T
    rows = ds.sample_rows(shots, seed=99, shot_offset=off)
    _, oev = oracle_run(oracle_lib, ds, shots, 99, off, nthreads=4, flips=False)
    assert np.array_equal(rows_unpack(rows, shots), rows_unpack(oev, shots))
    b8 = ds.sample(shots, seed=99, shot_offset=off)
    assert np.array_equal(b8_unpack(b8, ds.num_columns), rows_unpack(oev, shots))


@pytest.mark.parametrize("case", ["d3_p1e-2", "d5", "d9_highp"])
def test_error_model_sampler_equals_frame_sampler(oracle_lib, case):
    """The error-model sampler (kernel 4: detection events = XOR of the noise
    hits' output signatures) makes the frame sampler's own draws with one-word
    tiles: events (b8, rows) and counts agree bit for bit with the frame
    kernel and with the C oracle."""
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    text = _philox_cases()[case]
    dem = compile_detector_sampler(text, kernel=4)
    # one-word tiles and the error model's chunk lengths: the same draws
    frm = compile_detector_sampler(text, kernel=1, words_per_tile=1, fused_target_hits=2.0)
    assert dem.native.info["kernel"] == 4 and dem.tile_shots == 32 == frm.tile_shots
    for shots, off in ((4096, 0), (1000 + 7, 32 * 37)):
        a = dem.sample(shots, seed=11, shot_offset=off)
        assert np.array_equal(a, frm.sample(shots, seed=11, shot_offset=off))
        assert np.array_equal(dem.sample_rows(shots, seed=11, shot_offset=off),
                              frm.sample_rows(shots, seed=11, shot_offset=off))
        assert np.array_equal(dem.sample_counts(shots, seed=11, shot_offset=off),
                              b8_unpack(a, dem.num_columns).sum(axis=0))
    shots = 3 * 32 + 5
    _, oev = oracle_run(oracle_lib, dem, shots, 3, 64, nthreads=4, flips=False)
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
    frm = compile_detector_sampler(text, kernel=1, words_per_tile=1, fused_target_hits=2.0)
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
    frm = compile_detector_sampler(text, kernel=1, words_per_tile=1, fused_target_hits=2.0)
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
    frm = compile_detector_sampler(text, kernel=1, words_per_tile=1, fused_target_hits=2.0)
    for shots, off in ((2048, 0), (333, 32 * 9)):
        assert np.array_equal(dem.sample(shots, seed=4, shot_offset=off),
                              frm.sample(shots, seed=4, shot_offset=off))
        assert np.array_equal(dem.sample_rows(shots, seed=4, shot_offset=off),
                              frm.sample_rows(shots, seed=4, shot_offset=off))
