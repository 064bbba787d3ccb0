"""Kernel-level parity of the sm_100a kernels against the pinned CPU oracle (GPU box).

Every kernel that runs in the reference's rounding (laswp, trsm, panel, exact GEMM) must be
BITWISE equal to the oracle; the DMMA GEMM must match within the FP64 accumulation bound
|dC| <= 2 k u sum|a||b| (stated per test).
"""
import ctypes
import os

import numpy as np
import pytest

import oracle
from conftest import bitwise_equal

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def _lib():
    from paper_1804_07017_b200 import _lib

    return _lib


def _t(x, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def _stream():
    import torch

    return torch.cuda.current_stream().cuda_stream


def _sync():
    import torch

    torch.cuda.synchronize()


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (45, 38, 19), (128, 64, 16), (257, 131, 37), (1000, 700, 256),
                                   (300, 4, 5), (3, 500, 64)])
@pytest.mark.parametrize("exact", [True, False])
def test_gemm_update(cuda, m, n, k, exact):
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    c0 = rng.standard_normal((m, n))
    a0 = rng.standard_normal((m, k))
    b0 = rng.standard_normal((k, n))
    want = oracle.gemm_sub(c0.copy(), a0, b0)
    c, a, b = _t(c0, cuda), _t(a0, cuda), _t(b0, cuda)
    L = _lib().load()
    rc = L.pflu_gemm_update(c.data_ptr(), n, a.data_ptr(), k, b.data_ptr(), n, m, n, k, int(exact), _stream())
    _lib().check(rc, "gemm")
    got = c.cpu().numpy()
    if exact:
        assert bitwise_equal(got, want)
    else:
        bound = 2 * k * U * (np.abs(a0) @ np.abs(b0)) + 4 * U * np.abs(c0)
        assert np.all(np.abs(got - want) <= bound)


def test_gemm_update_tma_variant(cuda):
    """The TMA-fed GEMM (PFLU_GEMM_TMA=1: cp.async.bulk.tensor + mbarrier ring, permuted k quads)
    against the oracle, in a child process (the variant is chosen when libpflu loads)."""
    import subprocess
    import sys

    code = (
        "import sys, ctypes, numpy as np, torch; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');\n"
        "import oracle; from paper_1804_07017_b200 import _lib as lb; L = lb.load(); U = 2.0 ** -53\n"
        "for (m, n, k) in [(1000, 700, 256), (128, 64, 16), (3, 500, 64), (777, 130, 40), (4096, 512, 512)]:\n"
        "    r = np.random.default_rng(m + n + k); c0 = r.standard_normal((m, n)); a0 = r.standard_normal((m, k));"
        " b0 = r.standard_normal((k, n))\n"
        "    want = oracle.gemm_sub(c0.copy(), a0, b0)\n"
        "    c, a, b = (torch.from_numpy(x).cuda() for x in (c0, a0, b0))\n"
        "    lb.check(L.pflu_gemm_update(c.data_ptr(), n, a.data_ptr(), k, b.data_ptr(), n, m, n, k, 0,"
        " torch.cuda.current_stream().cuda_stream), 'gemm')\n"
        "    got = c.cpu().numpy(); bound = 2 * k * U * (np.abs(a0) @ np.abs(b0)) + 4 * U * np.abs(c0)\n"
        "    assert np.all(np.abs(got - want) <= bound), (m, n, k)\n"
        "print('tma ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PFLU_GEMM_TMA="1")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "tma ok" in out.stdout, out.stderr[-2000:]


def test_gemm_update_strided_unaligned(cuda):
    # odd leading dimensions and offsets force the 8-byte cp.async path
    rng = np.random.default_rng(3)
    big = rng.standard_normal((301, 211))
    want = big.copy()
    oracle.gemm_sub(want[40:301, 21:200], np.ascontiguousarray(want[40:301, 1:18]), np.ascontiguousarray(want[3:20, 21:200]))
    # oracle on views needs contiguous copies -> recompute directly
    want = big.copy()
    cv = want[40:301, 21:200].copy()
    oracle.gemm_sub(cv, big[40:301, 1:18].copy(), big[3:20, 21:200].copy())
    want[40:301, 21:200] = cv
    g = _t(big, cuda)
    L = _lib().load()
    base = g.data_ptr()
    ld = 211
    rc = L.pflu_gemm_update(base + (40 * ld + 21) * 8, ld, base + (40 * ld + 1) * 8, ld, base + (3 * ld + 21) * 8, ld,
                            261, 179, 17, 1, _stream())
    _lib().check(rc, "gemm")
    assert bitwise_equal(g.cpu().numpy(), want)


@pytest.mark.parametrize("nb,ncols", [(1, 5), (2, 3), (24, 37), (64, 1000), (256, 300), (512, 100), (130, 77)])
def test_trsm_bitwise(cuda, nb, ncols):
    rng = np.random.default_rng(nb + ncols)
    l0 = rng.standard_normal((nb, nb))
    x0 = rng.standard_normal((nb, ncols))
    want = oracle.trsm_llnu(l0, x0.copy())
    l, x = _t(l0, cuda), _t(x0, cuda)
    rc = _lib().load().pflu_trsm(l.data_ptr(), nb, nb, x.data_ptr(), ncols, ncols, _stream())
    _lib().check(rc, "trsm")
    assert bitwise_equal(x.cpu().numpy(), want)


def test_trsm_known_answer(cuda):
    # reference test_kernels.py:241-286: L=[[1,0],[2,1]], x=[1,0] -> [1,-2]; upper/diag ignored
    l = _t(np.array([[7.0, 9.0], [2.0, -3.0]]), cuda)
    x = _t(np.array([[1.0], [0.0]]), cuda)
    _lib().check(_lib().load().pflu_trsm(l.data_ptr(), 2, 2, x.data_ptr(), 1, 1, _stream()), "trsm")
    assert x.cpu().numpy().ravel().tolist() == [1.0, -2.0]


def test_trsm_golden(cuda, golden_small):
    l0, x0, want = golden_small["trsm__l"], golden_small["trsm__x"], golden_small["trsm__out"]
    l, x = _t(l0, cuda), _t(x0, cuda)
    nb, ncols = x0.shape
    _lib().check(_lib().load().pflu_trsm(l.data_ptr(), nb, nb, x.data_ptr(), ncols, ncols, _stream()), "trsm")
    assert bitwise_equal(x.cpu().numpy(), want)


def test_laswp_golden(cuda, golden_small):
    import torch

    x0, piv1, want = golden_small["laswp__a"], golden_small["laswp__piv1"], golden_small["laswp__out"]
    x = _t(x0, cuda)
    piv = torch.from_numpy(piv1 - 1).to(cuda)
    rc = _lib().load().pflu_laswp(x.data_ptr(), x0.shape[1], 0, x0.shape[1], piv.data_ptr(), 0, len(piv1), _stream())
    _lib().check(rc, "laswp")
    assert bitwise_equal(x.cpu().numpy(), want)


@pytest.mark.parametrize("seed,m,ncols,k1,k2", [(0, 50, 9, 0, 1), (1, 300, 200, 10, 90), (2, 2000, 33, 0, 512),
                                               (3, 5000, 700, 100, 356), (4, 1100, 64, 0, 1024)])
def test_laswp_random(cuda, seed, m, ncols, k1, k2):
    import torch

    rng = np.random.default_rng(seed)
    x0 = rng.standard_normal((m, ncols))
    piv0 = np.array([rng.integers(k, m) if rng.random() < 0.8 else k for k in range(k2)], dtype=np.int64)
    # repeated targets (collisions) on purpose
    if k2 - k1 > 4:
        piv0[k1 + 3] = piv0[k1 + 1] = max(piv0[k1 + 1], k1 + 3)
    want = oracle.laswp(x0.copy(), piv0, k1, k2)
    x = _t(x0, cuda)
    piv = torch.from_numpy(piv0).to(cuda)
    rc = _lib().load().pflu_laswp(x.data_ptr(), ncols, 0, ncols, piv.data_ptr(), k1, k2, _stream())
    _lib().check(rc, "laswp")
    assert bitwise_equal(x.cpu().numpy(), want)


def test_laswp_general_pivots(cuda):
    """Pivots below the current row (allowed by the reference laswp, kernels.py:273-300)."""
    import torch

    rng = np.random.default_rng(17)
    x0 = rng.standard_normal((300, 40))
    piv0 = np.array([rng.integers(0, 300) for _ in range(120)], dtype=np.int64)
    want = oracle.laswp(x0.copy(), piv0, 7, 120)
    x = _t(x0, cuda)
    piv = torch.from_numpy(piv0).to(cuda)
    _lib().check(_lib().load().pflu_laswp(x.data_ptr(), 40, 0, 40, piv.data_ptr(), 7, 120, _stream()), "laswp")
    assert bitwise_equal(x.cpu().numpy(), want)


def test_laswp_roundtrip_and_identity(cuda):
    # reference test_kernels.py:335-396: identity is a no-op; applying inverse swaps restores
    import torch

    rng = np.random.default_rng(9)
    x0 = rng.standard_normal((40, 24))
    x = _t(x0, cuda)
    ident = torch.arange(10, dtype=torch.int64, device=cuda)
    L = _lib().load()
    _lib().check(L.pflu_laswp(x.data_ptr(), 24, 0, 24, ident.data_ptr(), 0, 10, _stream()), "laswp")
    assert bitwise_equal(x.cpu().numpy(), x0)
    piv = torch.tensor([5, 7, 2, 39, 4], dtype=torch.int64, device=cuda)
    _lib().check(L.pflu_laswp(x.data_ptr(), 24, 0, 24, piv.data_ptr(), 0, 5, _stream()), "laswp")
    inv = oracle.laswp(x0.copy(), piv.cpu().numpy(), 0, 5)
    assert bitwise_equal(x.cpu().numpy(), inv)
    # undo: swaps in descending order are the inverse; express as ascending swaps of the reversed list
    y = x.cpu().numpy()
    for k in range(4, -1, -1):
        p = int(piv[k])
        y[[k, p]] = y[[p, k]]
    assert bitwise_equal(y, x0)


@pytest.mark.parametrize("m,w,ctas,leaf", [(64, 8, 0, 0), (300, 16, 0, 0), (1000, 64, 0, 0), (2048, 128, 3, 0),
                                          (5000, 256, 0, 0), (777, 100, 5, 8), (4096, 256, 16, 16),
                                          (20000, 256, 0, 0), (512, 512, 0, 0), (40, 40, 0, 32)])
@pytest.mark.parametrize("kernel", [1, 2, 3], ids=["grid", "cluster", "recursive"])
def test_panel_bitwise(cuda, m, w, ctas, leaf, kernel):
    """Recursive panel + cooperative leaf == lu_unb_run on the panel (exact op order)."""
    import torch
    from paper_1804_07017_b200 import _lib as lb

    rng = np.random.default_rng(m + w)
    p0 = rng.uniform(-1, 1, (m, w))
    want, wpiv, winfo = oracle.lu_unb(p0.copy())
    x = _t(p0, cuda)
    piv = torch.zeros(w, dtype=torch.int64, device=cuda)
    info = ctypes.c_int64(0)
    opt = lb.options(exact=True, panel_ctas=ctas if kernel != 2 else min(ctas, 16), leaf_width=leaf, panel_kernel=kernel)
    rc = lb.load().pflu_panel(x.data_ptr(), w, m, 0, 0, w, piv.data_ptr(), ctypes.byref(info), _stream(), ctypes.byref(opt))
    if kernel == 2 and rc == 3:
        pytest.skip("panel does not fit one cluster")
    lb.check(rc, "panel")
    assert np.array_equal(piv.cpu().numpy()[: len(wpiv)], wpiv)
    assert info.value == winfo
    assert bitwise_equal(x.cpu().numpy(), want)


@pytest.mark.parametrize("m,w,zero_cols", [(8192, 64, ()), (20000, 256, ()), (16500, 96, (0, 5, 6, 40)), (9000, 32, (31,)),
                                            (33000, 128, ())])
def test_panel_multicluster_bitwise(cuda, m, w, zero_cols):
    """Multi-cluster panel (panel_kernel 4: v2 exchange inside each 16-CTA cluster, one LL round between the
    clusters per column) == lu_unb_run on the panel, zero pivots included (_jit.py:154-187)."""
    import torch
    from paper_1804_07017_b200 import _lib as lb

    rng = np.random.default_rng(7 * m + w)
    p0 = rng.uniform(-1, 1, (m, w))
    for c in zero_cols:
        p0[:, c] = 0.0
    want, wpiv, winfo = oracle.lu_unb(p0.copy())
    for rep in range(3):
        x = _t(p0, cuda)
        piv = torch.zeros(w, dtype=torch.int64, device=cuda)
        info = ctypes.c_int64(0)
        opt = lb.options(exact=True, panel_kernel=lb.PANEL_MCLUSTER)
        lb.check(lb.load().pflu_panel(x.data_ptr(), w, m, 0, 0, w, piv.data_ptr(), ctypes.byref(info), _stream(),
                                      ctypes.byref(opt)), "panel")
        assert np.array_equal(piv.cpu().numpy()[: len(wpiv)], wpiv)
        assert info.value == winfo
        assert bitwise_equal(x.cpu().numpy(), want)


def test_panel_multicluster_special_values(cuda):
    """The multi-cluster exchange keeps the reference's pivot rules for special values (_jit.py:163-170): a NaN
    below the diagonal is never chosen, a NaN on the diagonal is kept, +-inf wins, exact ties go to the
    smallest row -- also when the tied rows sit in different clusters."""
    import warnings

    import torch
    from paper_1804_07017_b200 import _lib as lb

    m, w = 18000, 64
    p0 = np.random.default_rng(77).uniform(-1.0, 1.0, (m, w))
    p0[17000, 3] = np.nan
    p0[5, 5] = np.nan
    p0[16000, 20] = np.inf
    p0[9000, 30] = -np.inf
    p0[300, 40] = p0[12000, 40] = p0[17500, 40] = 9.0  # one tie across the clusters
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        want, wpiv, winfo = oracle.lu_unb(p0.copy())
    for exact in (True, False):
        x = _t(p0, cuda)
        piv = torch.zeros(w, dtype=torch.int64, device=cuda)
        info = ctypes.c_int64(0)
        opt = lb.options(exact=exact, panel_kernel=lb.PANEL_MCLUSTER)
        lb.check(lb.load().pflu_panel(x.data_ptr(), w, m, 0, 0, w, piv.data_ptr(), ctypes.byref(info), _stream(),
                                      ctypes.byref(opt)), "panel")
        assert np.array_equal(piv.cpu().numpy()[: len(wpiv)], wpiv), exact
        assert info.value == winfo
        if exact:
            assert np.array_equal(x.cpu().numpy(), want, equal_nan=True)


@pytest.mark.parametrize("m,w", [(300, 64), (5000, 256), (20000, 256), (2048, 512), (100, 200)])
def test_panel_recursive_dmma(cuda, m, w):
    """Recursive panel in DMMA mode: the oracle's pivots, factors within rounding of getf2's."""
    import torch
    from paper_1804_07017_b200 import _lib as lb

    p0 = np.random.default_rng(m * 3 + w).uniform(-1, 1, (m, w))
    want, wpiv, _ = oracle.lu_unb(p0.copy())
    x = _t(p0, cuda)
    piv = torch.zeros(w, dtype=torch.int64, device=cuda)
    info = ctypes.c_int64(0)
    opt = lb.options(exact=False, panel_kernel=lb.PANEL_RECURSIVE)
    lb.check(lb.load().pflu_panel(x.data_ptr(), w, m, 0, 0, w, piv.data_ptr(), ctypes.byref(info), _stream(),
                                  ctypes.byref(opt)), "panel")
    assert np.array_equal(piv.cpu().numpy()[: len(wpiv)], wpiv)
    assert info.value == 0
    assert np.max(np.abs(x.cpu().numpy() - want)) <= 1e-10


def test_panel_zero_column_info(cuda):
    import torch
    from paper_1804_07017_b200 import _lib as lb

    p0 = np.array([[1.0, 0.0, 2.0], [2.0, 0.0, 1.0], [4.0, 0.0, 3.0]])
    want, wpiv, winfo = oracle.lu_unb(p0.copy())
    x = _t(p0, cuda)
    piv = torch.zeros(3, dtype=torch.int64, device=cuda)
    info = ctypes.c_int64(0)
    rc = lb.load().pflu_panel(x.data_ptr(), 3, 3, 0, 0, 3, piv.data_ptr(), ctypes.byref(info), _stream(), None)
    lb.check(rc, "panel")
    assert info.value == 2 == winfo
    assert bitwise_equal(x.cpu().numpy(), want)
    assert np.all(x.cpu().numpy()[2:, 1] == 0.0)


def test_cli_sweep_with_check(cuda, capsys):
    """python -m paper_1804_07017_b200.cli --check on the reference's own instances."""
    from paper_1804_07017_b200 import cli

    assert cli.main(["--kind", "lu", "--strategy", "all", "--n-min", "300", "--n-max", "600", "--n-step", "300",
                     "--b", "64", "--reps", "1", "--check"]) == 0
    recs = cli.parse_csv(capsys.readouterr().out)
    assert len(recs) == 8 and {r.strategy for r in recs} == {"MTB", "LA", "LA_STATIC", "LA_MB"}
    for r in recs:
        assert r.gflops > 0 and 0 < r.residual <= 50      # reference test_factor.py:391-398 bound


@pytest.mark.parametrize("nb,ncols,d", [(256, 1000, 0), (256, 37, 300), (100, 300, 5), (33, 64, 0), (512, 40, 0), (512, 700, 3), (300, 200, 0)])
def test_swap_trsm_inv_matches_substitution(cuda, nb, ncols, d):
    """Fast-mode U12 solve (inverted 32x32 diagonal blocks + DMMA) == the substitution path up to
    rounding; pivots from a real partial-pivoting panel so the row interchanges are exercised."""
    import torch

    m = d + nb + 400
    rng = np.random.default_rng(nb + ncols + d)
    panel = rng.uniform(-1, 1, (m - d, nb))
    lu, piv, _ = oracle.lu_unb(panel.copy())  # |l| <= 1, pivots relative to row d
    full_piv = np.arange(m, dtype=np.int64)
    full_piv[d: d + nb] = np.asarray(piv[:nb], dtype=np.int64) + d
    a0 = rng.uniform(-1, 1, (m, ncols))
    l11 = _t(np.ascontiguousarray(lu[:nb, :nb]), cuda)
    L = _lib().load()
    dpiv = torch.from_numpy(full_piv).to(cuda)
    plan = torch.empty(1 + 3 * nb, dtype=torch.int64, device=cuda)
    _lib().check(L.pflu_pivot_plan(dpiv.data_ptr(), d, nb, plan.data_ptr(), _stream()), "plan")
    inv = torch.empty(((nb + 31) // 32) * 1024, dtype=torch.float64, device=cuda)
    _lib().check(L.pflu_diag_inv(l11.data_ptr(), nb, nb, inv.data_ptr(), _stream()), "diag_inv")
    x_sub, x_inv = _t(a0, cuda), _t(a0, cuda)
    _lib().check(L.pflu_swap_trsm_plan(x_sub.data_ptr(), ncols, d, nb, plan.data_ptr(), 0, ncols, l11.data_ptr(), nb,
                                       _stream()), "swap_trsm_plan")
    _lib().check(L.pflu_swap_trsm_inv(x_inv.data_ptr(), ncols, d, nb, plan.data_ptr(), 0, ncols, l11.data_ptr(), nb,
                                      inv.data_ptr(), _stream()), "swap_trsm_inv")
    ws, wi = x_sub.cpu().numpy(), x_inv.cpu().numpy()
    assert np.array_equal(ws[d + nb:], wi[d + nb:])  # rows below the block: swaps only, exact
    assert np.array_equal(ws[:d], wi[:d])
    top_s, top_i = ws[d: d + nb], wi[d: d + nb]
    assert np.abs(top_s - top_i).max() <= 1e-11 * max(1.0, np.abs(top_s).max())
