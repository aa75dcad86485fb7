"""libpfs.so on the CPU side: it loads, exports every symbol include/pfs.h
declares, and its host compiler (no GPU needed) behaves.  No compute calls."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2103_02202_b200 import _native as N
from paper_2103_02202_b200 import generators as gen
from paper_2103_02202_b200.program import flatten

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2103_02202_b200.build import build
    build()


def test_exports_match_header():
    with open(os.path.join(REPO, "include", "pfs.h")) as f:
        hdr = f.read()
    declared = set(re.findall(r"\b(pfs_[a-z_]+)\s*\(", hdr))
    assert declared == set(N.EXPORTS)
    L = ctypes.CDLL(N.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    assert N.lib().pfs_version() == 2


@pytest.mark.parametrize("cfg", [0, 1, 3])
def test_program_info_matches_survey_counts(cfg):
    f = flatten(gen.config_circuit(cfg))
    p = N.NativeProgram(f)
    info = p.info
    assert info["bframe_bits"] == {0: 708, 1: 75181, 3: 3700}[cfg]
    assert info["num_measurements"] == f.num_measurements
    assert info["num_columns"] == f.num_columns
    assert info["tile_shots"] == 32 * info["words_per_tile"]
    params, tab = p.noise_schedule()
    assert params.shape == (f.num_noise, 12)
    # every table is non-decreasing (inverse-CDF thresholds)
    for row in params:
        t = tab[row[5]:row[5] + row[6]]
        assert np.all(t[1:] >= t[:-1])


def test_d25_layout():
    f = flatten(gen.surface_code_memory(25, 25, 1e-3))
    p = N.NativeProgram(f)
    info = p.info
    assert info["bframe_bits"] == 518500
    assert info["smem_bytes"] <= 227 * 1024
    assert info["kernel"] == 1 and info["words_per_tile"] == 8 and info["groups"] == 2
    # every noise instruction rides inside its gate / collapse op; records stay
    # in x rows until the next reset spills them to the shared-memory ring
    assert info["fused_noise"] == f.num_noise and info["ring_in_smem"] == 1
    assert info["num_slots"] == 625  # one per measure qubit + the observable
    assert info["live_coin_rows"] == 0  # no coin reaches a detector of a Z memory
    assert info["num_ops"] < 250
    for W in (1, 2, 4, 8, 16):
        q = N.NativeProgram(f, words_per_tile=W, ring_in_smem=0, kernel=1)
        assert q.info["kernel"] == 1
        assert q.info["tile_shots"] == 32 * W and q.info["ring_in_smem"] == 0
    big = N.NativeProgram(flatten(gen.surface_code_memory(100, 2, 1e-3)))
    assert big.info["kernel"] == 1 and big.info["words_per_tile"] == 1 and big.info["ring_in_smem"] == 1


def test_binomial_thresholds_match_scipy():
    """The noise count table is the Binomial(L, p) inverse CDF in 2^-64 units."""
    from scipy.stats import binom

    f = flatten("X_ERROR(0.001) " + " ".join(map(str, range(64))) + "\n")
    p = N.NativeProgram(f, words_per_tile=8, ring_in_smem=0)
    params, tab = p.noise_schedule()
    L, cs, ca, nch, apps, tf, lf = (int(v) for v in params[0, :7])
    assert cs == min(L, 128) and ca == L // cs and nch == -(-apps // ca) * (256 // cs) and apps == 64
    cdf = binom.cdf(np.arange(lf), L, 0.001)
    got = tab[tf:tf + lf].astype(np.float64) / 2.0 ** 64
    assert np.allclose(got, cdf, rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_noise_schedule_matches_oracle_restatement(oracle_lib, cfg):
    """The product's chunk lengths follow the rule of DESIGN.md §4 (target 2
    hits per chunk); its geometry and Binomial tables
    equal the oracle's own (oracle/pfs_oracle.c computes them independently)."""
    from tests._util import rule_chunk_length

    f = flatten(gen.config_circuit(cfg))
    p = N.NativeProgram(f)
    params, tab = p.noise_schedule()
    params = params.astype(np.int64)
    T = p.tile_shots
    S = 32 * min(T // 32, 4)
    for row in f.instrs:
        if row[0] != 4:
            continue
        o = int(row[7])
        ar = 2 if row[1] == 4 else 1
        apps = int(row[2]) // ar
        mine = params[o]
        assert mine[0] == rule_chunk_length(float(f.noise_p[o]), apps, T, 2.0)
        ref, rtab = oracle_lib.noise_schedule_one(apps, int(row[1]), float(f.noise_p[o]), int(mine[0]), T, S)
        assert list(mine[[0, 1, 2, 3, 4, 6, 7, 8, 9]]) == list(ref[[0, 1, 2, 3, 4, 6, 7, 8, 9]])
        assert np.array_equal(tab[mine[5]:mine[5] + mine[6]], rtab)


def test_conflicting_instruction_is_split():
    # CX 0 1 1 2 must stay two sequential steps (frame_sim.py:61-62)
    f = flatten("CX 0 1 1 2\nM 0 1 2\n")
    p = N.NativeProgram(f)
    assert p.info["record_ops"] == 3
    assert p.info["num_ops"] == 2  # no detector reads the records: the event program drops M
    f2 = flatten("CX 0 1 2 3\nCX 4 5\nM 0 1 2 3 4 5\n")
    assert N.NativeProgram(f2).info["record_ops"] == 2  # merged CX, one M


def test_records_stay_in_x_rows_until_rewritten():
    # the M records live in x rows; R spills the one a later detector needs;
    # H rewrites x, so its record is spilled by a SPILL op before it
    f = flatten("R 0 1\nH 0\nCX 0 1\nM 0 1\nR 0\nH 1\nM 0 1\nDETECTOR rec[-2] rec[-4]\nDETECTOR rec[-1] rec[-3]\n")
    p = N.NativeProgram(f)
    assert p.info["num_slots"] == 2
    ops = p.ops()
    kinds = [int(k & 0xFF) for k in ops[:, 0]]
    assert 7 in kinds  # K_SPILL before the H on qubit 1


def test_errors_are_value_errors():
    f = flatten("H 0\nM 0\nDETECTOR rec[-1]\n")
    bad = flatten("H 0\nM 0\nDETECTOR rec[-1]\n")
    bad.instrs = bad.instrs.copy()
    bad.instrs[0, 2] = 5  # target range past the end
    with pytest.raises(ValueError):
        N.NativeProgram(bad)
    bad2 = flatten("X_ERROR(0.1) 0\n")
    bad2.noise_p = np.array([1.5])
    with pytest.raises(ValueError, match="noise probability"):
        N.NativeProgram(bad2)
    # a program whose frame table can never fit one CTA
    big = flatten("H 40000\n")
    with pytest.raises(ValueError, match="does not fit"):
        N.NativeProgram(big)
    p = N.NativeProgram(f)
    with pytest.raises(ValueError, match="num_shots must be >= 1"):
        p.run(N.MODE_DETECTORS, 0, 1, np.zeros(8, np.uint8), 8)


def test_oracle_not_reachable_from_product():
    """The product package must not import the oracle (it is the checker)."""
    pkg = os.path.join(REPO, "paper_2103_02202_b200")
    for root, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cpp", ".h")):
                with open(os.path.join(root, fn)) as f:
                    src = f.read()
                assert "import oracle" not in src and "from oracle" not in src, fn
                assert "pfs_oracle" not in src, fn


def test_error_model_sampler_scope():
    # the error-model sampler needs coin-independent outputs (QEC memories) and
    # produces detection events only
    from paper_2103_02202_b200 import generators as gen2
    p = N.NativeProgram(flatten(gen2.surface_code_memory(5, 5, 1e-3)), kernel=4)
    assert p.info["kernel"] == 4 and p.info["tile_shots"] == 32
    with pytest.raises(ValueError, match="measurement randomness"):
        N.NativeProgram(flatten(gen2.random_clifford(16, 20, 0.01, 1)), kernel=4)
