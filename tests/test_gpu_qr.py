"""Householder QR on the B200 (Kind.QR) against the reference and the oracle.

Parity bar (floating point; the reference's own block-reflector triangle T is formed with
numpy/BLAS products, so no bitwise mode exists for QR):
  * factors and tau: max|F_gpu - F_ref| / ||A||_max <= 1e-11 and |tau_gpu - tau_ref| <= 1e-11 against
    the reference's outputs (tests/golden/qr_cases.npz) and the pinned oracle (oracle.geqrf);
  * null reflectors exactly where the reference has them (tau == 0, column left unchanged);
  * backward error ||A - QR||_F / (n u ||A||_F) <= 10 and orthogonality ||Q^T Q - I||_F / (n u) <= 10
    (the reference's qr_residual, oracle.py:113-127; Q formed on the GPU by torch as the checker).
"""
import ctypes
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

TOL = 1e-11
GQ = np.load(os.path.join(GOLDEN, "qr_cases.npz"))


def _tags(prefix):
    return sorted({k.rsplit("_", 1)[0] for k in GQ.files if k.startswith(prefix)})


def _scaled_diff(f, g, a):
    return float(np.abs(np.asarray(f) - np.asarray(g)).max() / max(np.abs(a).max(), 1e-300))


def gpu_qr_residual(a0, f, tau):
    """(backward error, orthogonality) with Q = H_1 ... H_n formed by torch on the GPU (checker)."""
    import torch

    dev = torch.device("cuda:0")
    A = torch.from_numpy(np.ascontiguousarray(a0)).to(dev)
    F = torch.from_numpy(np.ascontiguousarray(f)).to(dev)
    T = torch.from_numpy(np.ascontiguousarray(tau)).to(dev)
    m, n = A.shape
    Q = torch.linalg.householder_product(torch.tril(F, -1) + torch.eye(m, n, device=dev, dtype=F.dtype), T)
    R = torch.triu(F[:n])
    u = 2.0 ** -53
    back = float(torch.linalg.norm(A - Q @ R) / (n * u * torch.linalg.norm(A)))
    orth = float(torch.linalg.norm(Q.T @ Q - torch.eye(n, device=dev, dtype=F.dtype)) / (n * u))
    return back, orth


@pytest.mark.parametrize("tag", _tags("mtb_") + _tags("la_"))
@pytest.mark.parametrize("lookahead", [0, 1])
def test_qr_matches_reference_golden(cuda, tag, lookahead):
    from paper_1804_07017_b200 import qr_factor

    a = GQ[f"{tag}_a"]
    f, tau = qr_factor(a.copy(), b=int(GQ[f"{tag}_b"]), lookahead=lookahead)
    assert _scaled_diff(f, GQ[f"{tag}_f"], a) <= TOL
    assert np.abs(tau - GQ[f"{tag}_tau"]).max() <= TOL
    assert np.array_equal(tau == 0.0, GQ[f"{tag}_tau"] == 0.0)
    back, orth = oracle.qr_residual(a, f, tau)
    assert back <= 10 and orth <= 10


def test_qr_dmf_drivers_return_qroutput(cuda):
    from paper_1804_07017_b200 import CacheConfig, Kind, Matrix, QrOutput, Strategy, dmf_la, dmf_mtb

    a = GQ["la_u64b16_a"]
    for drv, strat in ((dmf_la, Strategy.LA), (dmf_mtb, Strategy.MTB)):
        m = Matrix.from_array(a.copy())
        out = drv(m, CacheConfig(b=16), None, Kind.QR)
        assert isinstance(out, QrOutput) and out.strategy is strat and out.matrix is m
        assert _scaled_diff(m.array, GQ["la_u64b16_f"], a) <= TOL
        assert np.abs(out.tau - GQ["la_u64b16_tau"]).max() <= TOL


def test_zero_column_null_reflector(cuda):
    """A column that is zero below the diagonal gives tau = 0 and stays unchanged (_jit.py:203-205)."""
    from paper_1804_07017_b200 import qr_factor

    a = GQ["mtb_zerocol48b8_a"]
    f, tau = qr_factor(a.copy(), b=8, lookahead=1)
    ref_tau = GQ["mtb_zerocol48b8_tau"]
    assert np.array_equal(tau == 0.0, ref_tau == 0.0)
    a0 = np.zeros((3, 2))
    a0[:, 1] = [1.0, 2.0, 3.0]
    f0, t0 = qr_factor(a0.copy(), b=2)
    assert t0[0] == 0.0 and np.array_equal(f0[:, 0], a0[:, 0])


def _dev(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda:0")


@pytest.mark.parametrize("tag", _tags("unb_"))
def test_qr_panel_matches_reference_qr_unb(cuda, tag):
    from paper_1804_07017_b200 import _lib

    L = _lib.load()
    a = GQ[f"{tag}_a"]
    m, w = a.shape
    da = _dev(a.copy())
    dt = _dev(np.zeros(w))
    assert L.pflu_qr_panel(da.data_ptr(), w, m, 0, 0, w, dt.data_ptr(), None) == 0
    import torch

    torch.cuda.synchronize()
    assert _scaled_diff(da.cpu().numpy(), GQ[f"{tag}_f"], a) <= TOL
    assert np.abs(dt.cpu().numpy() - GQ[f"{tag}_tau"]).max() <= TOL


@pytest.mark.parametrize("m,w,d", [(4096, 64, 0), (40000, 32, 0), (3000, 100, 17), (70000, 48, 1000)])
def test_qr_panel_tall_multi_cta(cuda, m, w, d):
    """Panels tall enough to span many CTAs (grid exchange), leaves of 32 plus a ragged leaf, and a
    panel whose diagonal starts below row 0 (rows above d untouched)."""
    from paper_1804_07017_b200 import _lib
    import torch

    L = _lib.load()
    rng = np.random.default_rng(m + w)
    a = rng.uniform(-1, 1, (m, w + 3))
    da = _dev(a.copy())
    dt = _dev(np.zeros(w))
    assert L.pflu_qr_panel(da.data_ptr(), w + 3, m, d, 1, w, dt.data_ptr(), None) == 0
    torch.cuda.synchronize()
    got = da.cpu().numpy()
    ref, rtau = oracle.qr_unb(a[d:, 1:1 + w].copy())
    assert np.array_equal(got[:d], a[:d]) and np.array_equal(got[:, 0], a[:, 0])
    assert np.array_equal(got[:, w + 1:], a[:, w + 1:])
    assert _scaled_diff(got[d:, 1:1 + w], ref, a) <= 1e-10
    assert np.abs(dt.cpu().numpy() - rtau).max() <= 1e-10


def test_larft_and_block_reflector(cuda):
    from paper_1804_07017_b200 import _lib
    import torch

    L = _lib.load()
    rng = np.random.default_rng(5)
    mp, k, nc = 3000, 96, 500
    v, tau = oracle.qr_unb(rng.standard_normal((mp, k)))
    t_ref = oracle.larft(v, tau)
    dv, dtau = _dev(v), _dev(tau)
    dt = _dev(np.full((k, k), 7.0))
    assert L.pflu_larft(dv.data_ptr(), k, mp, k, dtau.data_ptr(), dt.data_ptr(), k, None) == 0
    t = dt.cpu().numpy()
    assert np.abs(t - t_ref).max() <= 1e-11 * max(1.0, np.abs(t_ref).max())
    assert np.all(np.tril(t, -1) == 0.0)
    c = rng.standard_normal((mp, nc))
    dc = _dev(c.copy())
    assert L.pflu_apply_block_reflector(dv.data_ptr(), k, mp, k, dtau.data_ptr(), dc.data_ptr(), nc, nc, None) == 0
    torch.cuda.synchronize()
    ref = c.copy()
    lib = oracle.lib()
    ptr = ctypes.POINTER(ctypes.c_double)
    vv = np.ascontiguousarray(v)
    lib.orc_apply_block_reflector(vv.ctypes.data_as(ptr), mp, k, k, t_ref.ctypes.data_as(ptr),
                                  ref.ctypes.data_as(ptr), nc, nc)
    assert _scaled_diff(dc.cpu().numpy(), ref, c) <= 1e-11


@pytest.mark.parametrize("m,n,b,lookahead", [(2048, 2048, 128, 1), (2048, 2048, 128, 0), (3000, 1000, 256, 1),
                                             (1100, 1000, 100, 1), (777, 513, 64, 0),
                                             # edge shapes: one column, b = 1, b > n, 1 x 1, odd b
                                             (5, 1, 4, 1), (20, 20, 1, 1), (33, 33, 64, 0), (1, 1, 1, 1),
                                             (100, 37, 7, 1), (64, 64, 64, 1)])
def test_qr_matches_oracle_medium(cuda, m, n, b, lookahead):
    from paper_1804_07017_b200 import qr_factor

    a = np.random.default_rng(m * 7 + n).uniform(-1, 1, (m, n))
    f, tau = qr_factor(a.copy(), b=b, lookahead=lookahead)
    ref, rtau = oracle.geqrf(a, b)
    assert _scaled_diff(f, ref, a) <= 1e-10
    assert np.abs(tau - rtau).max() <= 1e-10
    back, orth = gpu_qr_residual(a, f, tau)
    assert back <= 10 and orth <= 10


def test_qr_device_buffers_and_lookahead_agree(cuda):
    """Device-buffer entry point on the torch stream; depth 0 and 1 agree to rounding."""
    import torch
    from paper_1804_07017_b200 import qr_factor

    a = np.random.default_rng(2).standard_normal((8192, 8192))
    ta = _dev(a)
    f1, t1 = qr_factor(ta.clone(), b=256, lookahead=1)
    f0, t0 = qr_factor(ta.clone(), b=256, lookahead=0)
    torch.cuda.synchronize()
    assert float((f1 - f0).abs().max()) / float(ta.abs().max()) <= 1e-10
    back, orth = gpu_qr_residual(a, f1.cpu().numpy(), t1.cpu().numpy())
    assert back <= 10 and orth <= 10


def test_qr_deterministic_across_processes(cuda):
    """Every reduction (leaf exchanges, split-K slices) sums in a fixed order, so two runs in fresh
    processes give bitwise identical factors and tau."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, sys\n"
        "sys.path.insert(0, '.')\n"
        "from paper_1804_07017_b200 import qr_factor\n"
        "a = np.random.default_rng(4).uniform(-1, 1, (20000, 96))\n"
        "f, t = qr_factor(a, b=64, lookahead=1)\n"
        "np.save(sys.argv[1], np.concatenate([f.ravel(), t]))\n")
    outs = []
    for rep in range(2):
        path = os.path.join("/tmp", f"qr_det{rep}.npy")
        r = subprocess.run([sys.executable, "-c", code, path], cwd=root, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    assert outs[0].tobytes() == outs[1].tobytes()


def test_qr_cluster_and_grid_leaf_agree_bitwise(cuda):
    """PFLU_QR_CLUSTER=0 forces the cooperative-grid leaf kernel (global barrier + L2 exchange); the
    default uses one thread-block cluster (DSMEM exchange) for panels that fit.  With the same row
    split (panels <= 4096 rows: 256 rows per CTA in both) the sums run in the same order, so the
    factors must be bitwise identical."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, sys\n"
        "sys.path.insert(0, '.')\n"
        "from paper_1804_07017_b200 import qr_factor\n"
        "a = np.random.default_rng(6).uniform(-1, 1, (4000, 300))\n"
        "f, t = qr_factor(a, b=96, lookahead=1)\n"
        "np.save(sys.argv[1], np.concatenate([f.ravel(), t]))\n")
    outs = []
    for cl in ("0", "1"):
        path = os.path.join("/tmp", f"qr_cl{cl}.npy")
        env = dict(os.environ, PFLU_QR_CLUSTER=cl)
        r = subprocess.run([sys.executable, "-c", code, path], cwd=root, env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    assert outs[0].tobytes() == outs[1].tobytes()


def test_cli_qr_sweep_csv(cuda):
    """The reference-style bench CLI (python -m panelforge.bench --kind qr) on the B200: same CSV schema,
    backward error checked on the GPU."""
    import io

    from paper_1804_07017_b200 import cli

    recs = cli.run_sweep("qr", ["mtb", "la"], [256, 512], 64, 1, 0, True)
    assert [r.kind for r in recs] == ["QR"] * 4
    assert all(r.gflops > 0 and r.residual is not None and r.residual <= 10 for r in recs)
    buf = io.StringIO()
    cli.emit_csv(recs, buf)
    assert cli.parse_csv(buf.getvalue()) == recs


@pytest.mark.parametrize("lookahead", [0, 1])
def test_qr_trace_hook(cuda, lookahead):
    """QR trace records (factor.py:104-122): a PF per step (a chain), TU (depth 0) or TU_L / TU_R (depth 1)."""
    import torch
    from paper_1804_07017_b200 import geqrf_device

    n, b = 1000, 128
    a = torch.from_numpy(np.random.default_rng(21).uniform(-1, 1, (n, n))).cuda()
    tr = []
    geqrf_device(a, b, lookahead, trace=tr)
    steps = -(-n // b)
    pf = {e.k: e for e in tr if e.label == "PF"}
    assert sorted(pf) == list(range(steps))
    for k in range(1, steps):
        assert pf[k].start >= pf[k - 1].end - 1e-6
    for e in tr:
        assert 0.0 <= e.start <= e.end
    if lookahead == 0:
        assert sorted(e.k for e in tr if e.label == "TU") == list(range(steps - 1))
    else:
        assert sorted(e.k for e in tr if e.label == "TU_L") == list(range(steps - 1))
        assert sorted(e.k for e in tr if e.label == "TU_R") == list(range(steps - 2))


@pytest.mark.parametrize("kind_name", ["LU", "QR"])
def test_dmf_la_trace_like_reference(cuda, kind_name):
    """The reference's test_lookahead_overlap_instrumentation (test_factor.py:423-432) against the
    drop-in dmf_la: {PF, TU_R} among the labels and one PF per block."""
    from paper_1804_07017_b200 import CacheConfig, Kind, Matrix, dmf_la

    cfg = CacheConfig(b=64)
    n = 6 * cfg.b
    a0 = np.random.default_rng(22).random((n, n))
    m = Matrix.from_array(a0.copy())
    trace = []
    out = dmf_la(m, cfg, None, Kind[kind_name], malleable=True, trace=trace)
    labels = {ev.label for ev in trace}
    assert {"PF", "TU_R"} <= labels
    pf = {ev.k: ev for ev in trace if ev.label == "PF"}
    assert set(pf) == set(range(n // cfg.b))
    if kind_name == "QR":
        back, orth = oracle.qr_residual(a0, m.array, out.tau)
        assert back <= 10 and orth <= 10
    else:
        assert oracle.lu_residual(a0, m.array, out.pivots - 1) <= 10
