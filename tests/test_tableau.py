"""Native reference sample (csrc/pfs_tableau.cpp) against the reference's own
inverse-tableau simulator (`stabsim/tableau_sim.py`, SimState.run with
skip_noise=True — the body of `reference_sample`, lines 326-329).

The goldens `tests/golden/refsample_*.npz` were produced by the reference fed
a supplied collapse-coin stream (tests/golden/make_golden.py, gen_refsample);
the native simulator fed the same coins must reproduce every measurement bit
and every `determined_record` flag.  Host-only: no GPU needed.
"""

import glob
import os

import numpy as np
import pytest

from paper_2103_02202_b200 import generators as gen
from paper_2103_02202_b200 import tableau_sim as T
from paper_2103_02202_b200.circuit import as_circuit, detector_sets

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = sorted(os.path.basename(f)[10:-4] for f in glob.glob(os.path.join(HERE, "golden", "refsample_*.npz")))


def test_goldens_exist():
    assert len(CASES) >= 15


@pytest.mark.parametrize("name", CASES)
def test_bit_exact_vs_reference(name):
    z = np.load(os.path.join(HERE, "golden", f"refsample_{name}.npz"))
    bits, det, _ = T.reference_sample_with_coins(str(z["text"]), z["coins"])
    assert np.array_equal(bits, z["bits"])
    assert np.array_equal(det, z["determined"])


@pytest.mark.parametrize("d,r", [(3, 3), (5, 5), (11, 4)])
def test_surface_code_detectors_vanish_on_reference(d, r):
    # a reference sample is a valid noiseless outcome: every detector and the
    # observable (deterministic parities) is 0 for any coin stream
    text = gen.surface_code_memory(d, r, 1e-3)
    c = as_circuit(text)
    for seed in (0, 1, 2):
        ref = np.array(T.reference_sample(c, np.random.default_rng(seed)), dtype=np.uint8)
        assert len(ref) == c.num_measurements
        for s in detector_sets(c):
            assert int(ref[list(s)].sum()) % 2 == 0


def test_random_outcomes_follow_the_coins():
    # H then M: the single random measurement returns the coin
    for coin in (0, 1):
        bits, det, used = T.reference_sample_with_coins("H 0\nM 0\n", [coin])
        assert bits.tolist() == [coin] and det.tolist() == [0] and used == 1
    bits, det, _ = T.reference_sample_with_coins("X 0\nM 0\nMR 0\nM 0\n", [])
    assert bits.tolist() == [1, 1, 0] and det.tolist() == [1, 1, 1]


def test_errors():
    with pytest.raises(ValueError, match="coin stream exhausted"):
        T.reference_sample_with_coins("H 0 1\nM 0 1\n", [1])
    with pytest.raises(ValueError):
        T.reference_sample_with_coins("H 0\nM 0\n", [])
