"""Host-side API contracts of the drop-in (CPU): shapes, errors and record types mirror the
reference's dmf_la / dmf_mtb surface (pkg/src/panelforge/factor.py, core.py)."""
import numpy as np
import pytest

from paper_1804_07017_b200 import (CacheConfig, Kind, LuOutput, Matrix, Strategy, dmf_la, dmf_mtb, flops,
                                   lu_factor)


def test_flops_matches_reference_rounding():
    # reference factor.py:208-215: round(2 n^3 / 3), round(4 n^3 / 3)
    assert flops(Kind.LU, 1) == 1
    assert flops(Kind.LU, 2) == 5
    assert flops(Kind.LU, 32768) == round(2 * 32768 ** 3 / 3)
    assert flops(Kind.QR, 3) == 36
    with pytest.raises(ValueError):
        flops(Kind.LU, 0)


def test_wide_matrix_rejected():
    with pytest.raises(ValueError):
        lu_factor(np.zeros((4, 8)))
    with pytest.raises(ValueError):
        dmf_mtb(Matrix.zeros(4, 8), CacheConfig(b=16), None, Kind.LU)


def test_bad_arguments():
    with pytest.raises(ValueError):
        lu_factor(np.eye(4), lookahead=2)
    with pytest.raises(ValueError):
        lu_factor(np.eye(4), b=0)
    with pytest.raises(ValueError):
        CacheConfig(b=0)


def test_qr_bad_arguments():
    from paper_1804_07017_b200 import qr_factor

    with pytest.raises(ValueError):
        qr_factor(np.eye(4), lookahead=2)
    with pytest.raises(ValueError):
        qr_factor(np.eye(4), b=0)
    with pytest.raises(ValueError):
        qr_factor(np.zeros((3, 5)))   # wide: the reference rejects it (factor.py:293-297)


def test_matrix_container_is_column_major():
    a = np.arange(12.0).reshape(3, 4)
    m = Matrix.from_array(a)
    assert m.rows == 3 and m.cols == 4 and m.data.flags.f_contiguous
    assert np.array_equal(m.array, a)
    c = m.copy()
    c.array[0, 0] = -1
    assert m.array[0, 0] == 0


def test_output_record_fields():
    out = LuOutput(Matrix.zeros(2, 2), np.array([1, 2]), Strategy.LA, 0)
    assert out.strategy is Strategy.LA and out.info == 0 and list(out.pivots) == [1, 2]
