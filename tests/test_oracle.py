"""The C oracle, pinned against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import json
import os

import numpy as np
import pytest

from tests._util import (GOLDEN, b8_unpack, five_sigma, inject_cases, load_exact, load_inject,
                         load_noiseless, load_stats, pair_counts, rows_unpack, rule_chunk_lengths)


@pytest.mark.parametrize("name", inject_cases())
def test_oracle_injected_matches_reference(oracle_lib, name):
    from paper_2103_02202_b200.program import flatten

    O = oracle_lib
    text, B, coins, masks, flips_ref, events_ref = load_inject(name)
    prog = flatten(text)
    for T in sorted({32, 64, 256, B} & {t for t in (32, 64, 128, 256, 512, 1024) if t <= B or t == 32}):
        fl, ev = O.sample(prog, B, T, coins=coins, masks=masks, nthreads=2)
        assert np.array_equal(O.rows_to_b8(fl, B), flips_ref), (name, T)
        assert np.array_equal(O.rows_to_b8(ev, B), events_ref), (name, T)


def test_philox_known_answers(oracle_lib):
    # Random123 kat_vectors, philox4x32_10
    O = oracle_lib
    assert [hex(v) for v in O.philox([0, 0, 0, 0], [0, 0])] == \
        ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    assert [hex(v) for v in O.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2)] == \
        ["0x408f276d", "0x41c83b0e", "0xa20bc7c6", "0x6d5451fd"]
    assert [hex(v) for v in O.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
                                     [0xA4093822, 0x299F31D0])] == \
        ["0xd16cfe09", "0x94fdcceb", "0x5001e420", "0x24126ea1"]


@pytest.mark.parametrize("name", ["d3", "d5", "c1"])
def test_oracle_sampled_noise_matches_reference_statistics(oracle_lib, name):
    from paper_2103_02202_b200.program import flatten

    text, n_ref, counts_ref, pairs, pc_ref = load_stats(name)
    prog = flatten(text)
    shots = 1 << 16
    _, ev = oracle_lib.sample(prog, shots, 1024, seed=1234, flips=False, nthreads=8,
                              chunk_L=rule_chunk_lengths(prog, 1024, 0.5), vector_shots=128)
    bits = rows_unpack(ev, shots)
    assert five_sigma(bits.sum(axis=0), shots, counts_ref, n_ref) < 5.0
    assert five_sigma(pair_counts(bits, pairs), shots, pc_ref, n_ref) < 5.0


def test_oracle_detects_channel_transposition(oracle_lib):
    """Power check: swapping X_ERROR and Z_ERROR must fail 5 sigma."""
    from paper_2103_02202_b200.program import flatten

    text, n_ref, counts_ref, _, _ = load_stats("d5")
    bad = text.replace("X_ERROR", "Z_ERROR")
    prog = flatten(bad)
    shots = 1 << 16
    _, ev = oracle_lib.sample(prog, shots, 1024, seed=99, flips=False, nthreads=8,
                              chunk_L=rule_chunk_lengths(prog, 1024))
    bits = rows_unpack(ev, shots)
    assert five_sigma(bits.sum(axis=0), shots, counts_ref, n_ref) > 5.0


@pytest.mark.parametrize("name", ["d3", "d5", "c1", "mix"])
def test_oracle_noiseless(oracle_lib, name):
    from paper_2103_02202_b200.circuit import parse
    from paper_2103_02202_b200.program import flatten

    text, ref, det = load_noiseless(name)
    prog = flatten(text)
    shots = 2048
    fl, ev = oracle_lib.sample(prog, shots, 256, seed=5, nthreads=4, chunk_L=rule_chunk_lengths(prog, 256))
    flips = rows_unpack(fl, shots)
    assert not flips[:, det].any()
    if "DETECTOR" in text and name != "c1" and name != "mix":
        assert not rows_unpack(ev, shots).any()
    samples = flips ^ ref[None, :]
    assert np.array_equal(samples[:, det], np.broadcast_to(ref[det], samples[:, det].shape))


def _chi2_sf(stat, dof):
    from scipy.stats import chi2
    return float(chi2.sf(stat, dof))


def test_oracle_exact_tiny_distributions(oracle_lib):
    from paper_2103_02202_b200.program import flatten

    for case in load_exact():
        prog = flatten(case["text"])
        ref = np.array(case["reference"], dtype=np.uint8)
        shots = 20000
        fl, _ = oracle_lib.sample(prog, shots, 64, seed=17, events=False, chunk_L=rule_chunk_lengths(prog, 64, 0.5),
                                  vector_shots=32)
        samples = rows_unpack(fl, shots) ^ ref[None, :]
        keys = [tuple(r) for r in samples.tolist()]
        dist = {tuple(k): v for k, v in case["dist"]}
        obs = {}
        for k in keys:
            obs[k] = obs.get(k, 0) + 1
        assert set(obs) <= set(dist), set(obs) - set(dist)
        stat = sum((obs.get(k, 0) - shots * p) ** 2 / (shots * p) for k, p in dist.items())
        assert _chi2_sf(stat, max(1, len(dist) - 1)) > 1e-3, case["text"]


def test_frame_plans_match_reference():
    from paper_2103_02202_b200 import gates as G

    with open(os.path.join(GOLDEN, "frame_plans.json")) as f:
        ref = json.load(f)
    for name, rec in ref.items():
        g = G.GATE_MAP[name]
        assert g.kind == rec["kind"] and g.arity == rec["arity"], name
        if "frame_plan" in rec:
            mine = [[p, s, [list(x) for x in src]] for p, s, src in g.frame_plan]
            assert mine == rec["frame_plan"], name
        if "noise_patterns" in rec:
            assert [list(p) for p in g.noise_patterns] == rec["noise_patterns"], name
        assert g.records == rec["records"] and g.resets == rec["resets"]


def test_b8_known_answers(oracle_lib):
    """shot [1,0,0,0,0,0,0,0,1] -> 0x01 0x01; padding zero."""
    rows = np.zeros((9, 1), dtype=np.uint32)
    rows[0, 0] = 1
    rows[8, 0] = 1
    out = oracle_lib.rows_to_b8(rows, 1)
    assert out.tolist() == [[1, 1]]


@pytest.mark.parametrize("layout", [(1024, 128, 2.0), (256, 128, 0.5), (32, 32, 2.0), (64, 64, 0.25)])
def test_oracle_statistics_do_not_depend_on_layout(oracle_lib, layout):
    """Tile size, vector size and chunk length choose the draw order only: the
    event statistics match the reference's at every layout (d=3, p=1e-2)."""
    from paper_2103_02202_b200.program import flatten

    T, S, target = layout
    text, n_ref, counts_ref, pairs, pc_ref = load_stats("d3")
    prog = flatten(text)
    shots = 1 << 16
    _, ev = oracle_lib.sample(prog, shots, T, seed=4321, flips=False, nthreads=8,
                              chunk_L=rule_chunk_lengths(prog, T, target), vector_shots=S)
    bits = rows_unpack(ev, shots)
    assert five_sigma(bits.sum(axis=0), shots, counts_ref, n_ref) < 5.0
    assert five_sigma(pair_counts(bits, pairs), shots, pc_ref, n_ref) < 5.0


@pytest.mark.parametrize("p", [1e-3, 5e-3, 0.01, 0.2, 0.7])
@pytest.mark.parametrize("L", [1, 64, 512, 2048])
def test_oracle_binomial_tables_match_scipy(oracle_lib, p, L):
    """The oracle's own count tables are the Binomial(L, p) inverse CDF in
    2^-64 units (entropy.py's Bernoulli(p) trials, counted per chunk)."""
    from scipy.stats import binom

    if L * p > 40:
        pytest.skip("chunks of this length are never chosen for this p (mean hits <= 2)")
    params, tab = oracle_lib.noise_schedule_one(1000, 3, p, L, 256, 128)
    params = [int(v) for v in params]
    assert params[0] == L and params[1] == min(L, 128) and params[2] == L // min(L, 128)
    assert params[3] == -(-1000 // params[2]) * (256 // params[1])
    cdf = binom.cdf(np.arange(len(tab)), L, p)
    got = tab.astype(np.float64) / 2.0 ** 64
    assert np.allclose(got, cdf, rtol=1e-9, atol=1e-15)
    assert np.all(tab[1:] >= tab[:-1])
    # the thresholds stop where the upper tail drops below 2^-64 (or at count L)
    assert binom.sf(len(tab) - 1, L, p) < 1e-12 or len(tab) >= L


def test_oracle_rows_to_b8_threads_agree(oracle_lib):
    rng = np.random.default_rng(3)
    rows = rng.integers(0, 2 ** 32, size=(77, 40), dtype=np.uint64).astype(np.uint32)
    xor = rng.integers(0, 2, size=77, dtype=np.uint8)
    shots = 40 * 32 - 5
    ref = np.packbits(rows_unpack(rows, shots) ^ xor[None, :], axis=1, bitorder="little")
    for nt in (1, 3, 8):
        assert np.array_equal(oracle_lib.rows_to_b8(rows, shots, xor, nthreads=nt), ref)
    # power-of-two row pitch, whole 512-shot chunks, rows a multiple of 8, no xor
    rows = rng.integers(0, 2 ** 32, size=(64, 64), dtype=np.uint64).astype(np.uint32)
    ref = np.packbits(rows_unpack(rows, 2048), axis=1, bitorder="little")
    for nt in (1, 5):
        assert np.array_equal(oracle_lib.rows_to_b8(rows, 2048, nthreads=nt), ref)
