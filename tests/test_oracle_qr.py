"""QR oracle (oracle/pflu_oracle.c orc_qr_*) pinned against the reference's own outputs
(tests/golden/qr_cases.npz, made by tests/golden/make_golden_qr.py from the unmodified reference).

The panel (qr_unb, reference _jit.py:190-218) is pinned BITWISE.  The blocked factorization's
block-reflector triangle T comes from numpy/BLAS products in the reference (factor.py:174-189),
so the blocked factors agree to rounding: max|F - F_ref| / ||A||_max <= 1e-13."""
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "qr_cases.npz")


@pytest.fixture(scope="module")
def gq():
    return np.load(GOLD)


def _tags(prefix):
    return sorted({k.rsplit("_", 1)[0] for k in np.load(GOLD).files if k.startswith(prefix)})


@pytest.mark.parametrize("tag", _tags("unb_"))
def test_qr_unb_bitwise_reference(gq, tag):
    f, tau = oracle.qr_unb(gq[f"{tag}_a"].copy())
    assert f.tobytes() == np.ascontiguousarray(gq[f"{tag}_f"]).tobytes()
    assert tau.tobytes() == gq[f"{tag}_tau"].tobytes()


@pytest.mark.parametrize("tag", _tags("mtb_") + _tags("la_"))
def test_geqrf_matches_reference(gq, tag):
    a = gq[f"{tag}_a"]
    f, tau = oracle.geqrf(a, int(gq[f"{tag}_b"]))
    scale = np.abs(a).max()
    assert np.abs(f - gq[f"{tag}_f"]).max() / scale <= 1e-13
    assert np.abs(tau - gq[f"{tag}_tau"]).max() <= 1e-13
    # the zero column of the singular case gives tau = 0 exactly, like the reference
    assert np.array_equal(tau == 0.0, gq[f"{tag}_tau"] == 0.0)
    factor, ortho = oracle.qr_residual(a, f, tau)
    assert factor <= 10 and ortho <= 10


def test_larft_identity():
    a = np.random.default_rng(3).standard_normal((40, 12))
    f, tau = oracle.qr_unb(a.copy())
    t = oracle.larft(f, tau)
    v = np.tril(f, -1)
    np.fill_diagonal(v, 1.0)
    h = np.eye(40)
    for j in range(12):
        h = h @ (np.eye(40) - tau[j] * np.outer(v[:, j], v[:, j]))
    assert np.abs(h - (np.eye(40) - v @ t @ v.T)).max() < 1e-14


def test_block_size_invariance_to_rounding():
    a = np.random.default_rng(8).uniform(-1, 1, (96, 96))
    f1, t1 = oracle.geqrf(a, 96)
    f2, t2 = oracle.geqrf(a, 16)
    assert np.abs(f1 - f2).max() < 1e-13 and np.abs(t1 - t2).max() < 1e-13
    fu, tu = oracle.qr_unb(a.copy())
    assert f1.tobytes() == fu.tobytes() and t1.tobytes() == tu.tobytes()
