"""The drop-in entry points (collect_flips / sample_batch / detector_events /
sample_detection_events) on the GPU, against the reference's contracts."""

import numpy as np
import pytest

from tests._util import b8_unpack, load_inject, load_noiseless

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_collect_flips_and_detector_events_compose():
    from paper_2103_02202_b200 import frame_sim, generators as gen
    from paper_2103_02202_b200.circuit import detector_and_observable_sets, parse
    from paper_2103_02202_b200.io_formats import detector_events

    text = gen.surface_code_memory(5, 5, 5e-3)
    c = parse(text)
    flips = frame_sim.collect_flips(c, 3000, np.random.default_rng(1))
    assert flips.num_shots == 3000 and flips.num_results == c.num_measurements
    ev = detector_events(flips, detector_and_observable_sets(c))
    # detector_events on the GPU equals the XOR definition computed on the host
    fm = flips.to_numpy()
    expect = np.stack([np.bitwise_xor.reduce(fm[:, list(s)], axis=1)
                       for s in detector_and_observable_sets(c)], axis=1)
    assert np.array_equal(ev.to_numpy(), expect)
    # the fused device path gives the same events for the same seed stream
    fused = frame_sim.sample_detection_events(c, 3000, np.random.default_rng(1))
    assert fused.num_results == len(detector_and_observable_sets(c))


def test_detector_events_errors():
    from paper_2103_02202_b200.io_formats import SampleTable, detector_events
    t = SampleTable.from_numpy(np.zeros((4, 3), np.uint8))
    with pytest.raises(ValueError, match="detector 0 references measurement 5, have 3"):
        detector_events(t, [(5,)])
    assert detector_events(t, []).num_results == 0


def test_sample_batch_noiseless_equals_reference():
    from paper_2103_02202_b200 import frame_sim
    text, ref, det = load_noiseless("d5")
    out = frame_sim.sample_batch(text, ref, 2000, np.random.default_rng(3))
    s = out.to_numpy()
    assert np.array_equal(s[:, det], np.broadcast_to(ref[det], s[:, det].shape))
    with pytest.raises(ValueError, match="reference has 3 bits, circuit measures"):
        frame_sim.sample_batch(text, [0, 1, 0], 10, np.random.default_rng(0))


def test_error_conventions():
    from paper_2103_02202_b200 import frame_sim
    with pytest.raises(ValueError, match="num_shots must be >= 1"):
        frame_sim.collect_flips("M 0\n", 0, np.random.default_rng(0))
    with pytest.raises(ValueError, match="batch_size must be >= 1"):
        frame_sim.collect_flips("M 0\n", 5, np.random.default_rng(0), batch_size=0)


def test_h_m_is_fair():
    """`H 0; M 0` gives 0.5 +- 0.02 at 10^4 shots."""
    from paper_2103_02202_b200 import frame_sim
    out = frame_sim.sample_batch("H 0\nM 0\n", [0], 10000, np.random.default_rng(7))
    assert abs(out.to_numpy().mean() - 0.5) < 0.02


def test_reference_circuit_objects_accepted():
    """A reference `stabsim` Circuit is accepted wherever a circuit is (the
    pip-installed copy in baseline/_ref travels to the GPU box)."""
    import os
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for cand in (os.path.join(repo, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(cand, "stabsim")):
            sys.path.insert(0, cand)
            break
    else:
        pytest.skip("reference package not installed (baseline/_ref) or mounted")
    from stabsim import circuit as rc
    from paper_2103_02202_b200 import frame_sim
    c = rc.parse("H 0\nCNOT 0 1\nM 0 1\nDETECTOR rec[-1] rec[-2]\n")
    ev = frame_sim.sample_detection_events(c, 500, np.random.default_rng(0))
    assert not ev.to_numpy().any()


def test_compile_sampler_native_reference():
    # compile_sampler without a reference computes the native inverse-tableau
    # reference sample (tableau_sim.py): noiseless samples keep every detector
    # parity at 0, and records whose flips are always 0 (Z-type stabilizers
    # here: every Z ancilla round) equal the reference
    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.circuit import as_circuit, detector_sets
    from paper_2103_02202_b200.sampler import compile_sampler

    text = gen.surface_code_memory(5, 5, 0.0)
    c = as_circuit(text)
    s = compile_sampler(c, seed=3)
    smp = b8_unpack(s.sample(2048, seed=9), c.num_measurements)
    ref = s.reference
    fixed = np.all(smp == smp[0], axis=0)  # shot-invariant records
    assert fixed.sum() > c.num_measurements // 4
    assert np.array_equal(smp[0, fixed], ref[fixed])
    for ds in detector_sets(c):
        assert not np.any(smp[:, list(ds)].sum(axis=1) % 2)


@pytest.mark.parametrize("R", [1, 7, 8, 31, 33, 255, 256, 300, 1023, 2000])
@pytest.mark.parametrize("density", [0.0, 0.002, 0.05, 0.5, 1.0])
def test_device_writers_match_reference_formats(R, density):
    # write_table on the GPU (01 / hits / r8) equals the host writers, which are
    # byte-exact with the reference's (io_formats.py:66-187)
    from paper_2103_02202_b200.io_formats import SampleTable, write_table, write_table_device

    rng = np.random.default_rng(R * 7 + int(density * 1000))
    shots = 97
    mat = (rng.random((shots, R)) < density).astype(np.uint8)
    t = SampleTable.from_numpy(mat)
    for fmt in ("01", "hits", "r8", "b8"):
        assert write_table_device(t.b8, R, fmt) == write_table(t, fmt), fmt


def test_device_writers_on_sampled_events():
    import torch
    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.io_formats import SampleTable, write_table, write_table_device
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    ds = compile_detector_sampler(gen.surface_code_memory(9, 9, 5e-3))
    nb = (ds.num_columns + 7) // 8
    dev = torch.empty((5000, nb), dtype=torch.uint8, device="cuda")
    ds.sample(5000, seed=1, out=dev)
    host = dev.cpu().numpy()
    t = SampleTable.from_b8(host, ds.num_columns)
    for fmt in ("hits", "r8", "01"):
        assert write_table_device(dev, ds.num_columns, fmt) == write_table(t, fmt)


@pytest.mark.parametrize("d,shots,offset_tiles", [(5, 1 << 21, 0), (25, 1 << 19, 0), (25, (1 << 19) + 12345, 3)])
def test_frame_transpose_pipeline_bit_exact(d, shots, offset_tiles):
    """The pipelined launch (frame kernel of sub-chunk i+1 on a high-priority
    stream while the transpose of sub-chunk i drains on another) gives the same
    events as one frame launch then one transpose, with any sub-chunk count and
    thread count."""
    import torch
    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    text = gen.surface_code_memory(d, d, 2e-3)
    s1 = compile_detector_sampler(text, pipeline=1)
    nb = (s1.num_columns + 7) // 8
    off = offset_tiles * s1.info["tile_shots"]
    dev = torch.empty((shots, nb), dtype=torch.uint8, device="cuda")
    s1.sample(shots, seed=77, out=dev, shot_offset=off)
    torch.cuda.synchronize()
    ref = dev.cpu().numpy()
    for pipe, thr in ((0, 0), (3, 512), (7, 0)):
        dev.zero_()
        compile_detector_sampler(text, pipeline=pipe, threads=thr).sample(shots, seed=77, out=dev, shot_offset=off)
        torch.cuda.synchronize()
        assert np.array_equal(dev.cpu().numpy(), ref), (pipe, d)
    # host output (chunked D2H) and counts over the same launch path
    assert np.array_equal(compile_detector_sampler(text).sample(shots, seed=77, shot_offset=off), ref)
    cr = s1.sample_counts(shots, seed=77, shot_offset=off)
    cp = compile_detector_sampler(text, pipeline=4).sample_counts(shots, seed=77, shot_offset=off)
    assert np.array_equal(np.asarray(cp), np.asarray(cr))
    assert int(np.asarray(cr, dtype=np.int64).sum()) == int(np.unpackbits(ref, axis=1).sum())
