"""Output formats and SampleTable (host side), pinned to the SPEC's known
answers and to byte-exact round trips."""

import numpy as np
import pytest

from paper_2103_02202_b200 import io_formats as F
from paper_2103_02202_b200.io_formats import SampleTable


def test_b8_known_answers():
    t = SampleTable.from_numpy(np.array([[1, 0, 0, 0, 0, 0, 0, 0, 1]]))
    assert F.write_b8(t) == bytes([0x01, 0x01])
    assert F.write_b8(SampleTable.from_numpy(np.zeros((1, 8), np.uint8))) == b"\x00"
    assert F.write_b8(SampleTable.from_numpy(np.ones((1, 8), np.uint8))) == b"\xff"


def test_hits_and_r8_known_answers():
    t = SampleTable.from_numpy(np.array([[0, 1, 0, 1]]))
    assert F.write_hits(t) == b"1,3\n"
    assert F.write_r8(SampleTable.from_numpy(np.zeros((1, 3), np.uint8))) == b"\x03"
    assert F.write_r8(SampleTable.from_numpy(np.zeros((1, 300), np.uint8))) == b"\xff\x2d"
    assert F.write_01(SampleTable.from_numpy(np.array([[1], [0]]))) == b"1\n0\n"


@pytest.mark.parametrize("fmt", ["01", "b8", "hits", "r8"])
@pytest.mark.parametrize("shape", [(1, 1), (7, 9), (33, 300), (5, 1000), (3, 8)])
def test_round_trip(fmt, shape):
    rng = np.random.default_rng(shape[0] * 1000 + shape[1])
    mat = (rng.random(shape) < 0.2).astype(np.uint8)
    t = SampleTable.from_numpy(mat)
    data = F.write_table(t, fmt)
    back = F.FORMATS[fmt][1](data) if fmt == "01" else F.FORMATS[fmt][1](data, shape[1])
    assert np.array_equal(back.to_numpy(), mat)


def test_sampletable_views_agree():
    rng = np.random.default_rng(0)
    mat = (rng.random((17, 23)) < 0.5).astype(np.uint8)
    t = SampleTable.from_numpy(mat)
    assert t.get(3, 5) == mat[3, 5]
    assert t.row(4).bits == int("".join(map(str, mat[4][::-1])), 2)
    rows = SampleTable.from_rows(t.bits.rows, 23)
    assert rows == t
    assert np.array_equal(SampleTable.from_b8(t.b8, 23).to_numpy(), mat)
    with pytest.raises(ValueError):
        F.write_table(t, "nope")


def test_reference_formats_byte_exact():
    """Our writers vs the reference writers on the same table (skipped when the
    reference is not mounted, e.g. on the GPU box)."""
    import os
    import sys
    if not os.path.isdir("/root/reference/pkg/src"):
        pytest.skip("reference not mounted")
    sys.path.insert(0, "/root/reference/pkg/src")
    from stabsim import io_formats as R
    rng = np.random.default_rng(5)
    mat = (rng.random((20, 530)) < 0.05).astype(np.uint8)
    rt = R.SampleTable.from_numpy(mat)
    ot = SampleTable.from_numpy(mat)
    for fmt in ("01", "b8", "hits", "r8"):
        assert R.write_table(rt, fmt) == F.write_table(ot, fmt), fmt
