"""End-to-end parity of the B200 factorization with the reference (GPU box).

* exact mode (reference rounding everywhere) must be BITWISE equal to the reference's own
  output: small cases from tests/golden/small_cases.npz and the full C1/C2/C3 factors via the
  sha256 the reference produced (tests/golden/configs.json, made by make_golden.py);
* DMMA mode (default) must give the SAME pivots (north_star: identical except top-two ties within
  1e-12 relative -- none occur on these inputs), ||PA-LU||_F/(||A||_F n eps) <= 10 and
  max|LU_gpu - LU_ref| / ||A||_max <= 10 (we also assert a much tighter 1e-8 on the latter).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, bitwise_equal

pytestmark = pytest.mark.gpu

CONFIGS = json.load(open(os.path.join(GOLDEN, "configs.json")))
PIVOTS = np.load(os.path.join(GOLDEN, "configs_pivots.npz"))


def config_matrix(name):
    if name == "c1":
        return np.random.default_rng(0).uniform(-1.0, 1.0, size=(2048, 2048))
    if name in ("c2", "c2s"):
        a = np.random.default_rng(1).uniform(-1.0, 1.0, size=(8192, 8192))
        if name == "c2s":
            a[np.diag_indices(8192)] += 8192.0
        return a
    if name == "c3":
        return np.random.default_rng(2).standard_normal((16384, 16384))
    if name == "c4":
        return np.random.default_rng(3).uniform(-1.0, 1.0, size=(32768, 32768))
    raise KeyError(name)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gpu_residual(a0, lu, piv, block=4096):
    """||PA - LU||_F / (||A||_F n u) on the GPU (torch fp64 matmul as the checker only)."""
    import torch

    dev = torch.device("cuda:0")
    n = a0.shape[1]
    perm = oracle.perm_from_pivots(piv, a0.shape[0])
    U_ = torch.triu(torch.from_numpy(np.ascontiguousarray(lu[:n])).to(dev))
    err2 = 0.0
    for r0 in range(0, a0.shape[0], block):
        r1 = min(a0.shape[0], r0 + block)
        Lb = torch.from_numpy(np.ascontiguousarray(lu[r0:r1, :n])).to(dev)
        Lb = torch.tril(Lb, diagonal=r0 - 1)   # global (i, j) kept iff j < i
        idx = torch.arange(r0, min(r1, n), device=dev)
        Lb[idx - r0, idx] = 1.0
        d = torch.from_numpy(np.ascontiguousarray(a0[perm[r0:r1]])).to(dev) - Lb @ U_
        err2 += float((d * d).sum())
        del Lb, d
    return np.sqrt(err2) / (n * oracle.UNIT_ROUNDOFF * np.linalg.norm(a0))


def run(a0, b, lookahead, exact, panel_kernel=0):
    from paper_1804_07017_b200 import lu_factor

    lu, piv, info = lu_factor(a0.copy(), b=b, lookahead=lookahead, exact=exact, return_info=True,
                              panel_kernel=panel_kernel)
    return lu, piv, info


SMALL = ["swap2", "diag4", "zero3", "grid16", "grid32", "grid80", "grid97", "u300", "n200", "tall57x32",
         "sing48", "la6b", "la4b7", "n257b64", "tie4"]


@pytest.mark.parametrize("tag", SMALL)
@pytest.mark.parametrize("lookahead", [0, 1])
def test_small_golden_exact(cuda, golden_small, tag, lookahead):
    a0 = golden_small[f"{tag}__a"]
    b, info, _ = golden_small[f"{tag}__meta"]
    with np.errstate(all="ignore"):
        import warnings

        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            lu, piv, inf = run(a0, int(b), lookahead, exact=True)
    assert inf == info
    assert np.array_equal(piv, golden_small[f"{tag}__piv"])
    assert bitwise_equal(lu, golden_small[f"{tag}__f"])


@pytest.mark.parametrize("tag", ["u300", "n200", "grid97", "n257b64", "la6b"])
@pytest.mark.parametrize("b", [16, 64, 256])
def test_small_dmma(cuda, golden_small, tag, b):
    a0 = golden_small[f"{tag}__a"]
    lu, piv, inf = run(a0, b, 1, exact=False)
    assert np.array_equal(piv, golden_small[f"{tag}__piv"])
    assert oracle.lu_residual(a0, lu, piv) <= 10
    assert oracle.max_rel_diff(lu, golden_small[f"{tag}__f"], a0) <= 1e-10


@pytest.mark.parametrize("lookahead", [0, 1])
def test_c1_exact_matches_reference_sha(cuda, lookahead):
    a0 = config_matrix("c1")
    lu, piv, info = run(a0, 128, lookahead, exact=True)
    assert info == 0
    assert np.array_equal(piv, PIVOTS["c1"])
    assert sha(lu) == CONFIGS["c1"]["sha256_factors"]


@pytest.mark.parametrize("lookahead", [0, 1])
def test_c1_recursive_panel(cuda, lookahead):
    """Every step's panel on the recursive panel (panel_kernel 3): exact mode keeps the reference's
    bitwise factors, DMMA mode its pivots."""
    a0 = config_matrix("c1")
    lu, piv, info = run(a0, 128, lookahead, exact=True, panel_kernel=3)
    assert info == 0 and np.array_equal(piv, PIVOTS["c1"])
    assert sha(lu) == CONFIGS["c1"]["sha256_factors"]
    lu2, piv2, _ = run(a0, 256, lookahead, exact=False, panel_kernel=3)
    assert np.array_equal(piv2, PIVOTS["c1"])
    assert gpu_residual(a0, lu2, piv2) <= 10
    assert oracle.max_rel_diff(lu2, lu, a0) <= 1e-8


@pytest.mark.parametrize("tag", SMALL)
def test_small_golden_recursive_panel(cuda, golden_small, tag):
    a0 = golden_small[f"{tag}__a"]
    b, info, _ = golden_small[f"{tag}__meta"]
    import warnings

    with np.errstate(all="ignore"), warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        lu, piv, inf = run(a0, int(b), 1, exact=True, panel_kernel=3)
    assert inf == info
    assert np.array_equal(piv, golden_small[f"{tag}__piv"])
    assert bitwise_equal(lu, golden_small[f"{tag}__f"])


@pytest.mark.parametrize("lookahead", [0, 1])
def test_c1_dmma(cuda, lookahead):
    a0 = config_matrix("c1")
    ref, rpiv, _ = oracle.getrf(a0, 128)
    assert sha(ref) == CONFIGS["c1"]["sha256_factors"]      # oracle still pinned
    lu, piv, info = run(a0, 128, lookahead, exact=False)
    assert np.array_equal(piv, PIVOTS["c1"])
    assert gpu_residual(a0, lu, piv) <= 10
    assert oracle.max_rel_diff(lu, ref, a0) <= 1e-8


@pytest.mark.parametrize("name", ["c2", "c2s"])
def test_c2(cuda, name):
    a0 = config_matrix(name)
    lu, piv, info = run(a0, 256, 1, exact=False)
    assert np.array_equal(piv, PIVOTS[name])
    if name == "c2s":
        assert np.array_equal(piv, np.arange(8192))          # no row swaps in the shifted variant
    assert gpu_residual(a0, lu, piv) <= 10
    lu_x, piv_x, _ = run(a0, 256, 1, exact=True)
    assert sha(lu_x) == CONFIGS[name]["sha256_factors"]
    assert sha(lu[:256]) != "" and oracle.max_rel_diff(lu, lu_x, a0) <= 1e-8


@pytest.mark.parametrize("b", [64, 128, 256, 512])
def test_c3_block_sweep(cuda, b):
    a0 = config_matrix("c3")
    for lookahead in (0, 1):
        lu, piv, info = run(a0, b, lookahead, exact=False)
        assert np.array_equal(piv, PIVOTS["c3"]), (b, lookahead)
        if b == 256:
            assert gpu_residual(a0, lu, piv) <= 10
    lu_x, piv_x, _ = run(a0, b, 1, exact=True)
    assert sha(lu_x) == CONFIGS["c3"]["sha256_factors"]
    assert oracle.max_rel_diff(lu, lu_x, a0) <= 1e-8


@pytest.mark.parametrize("lookahead", [0, 1])
def test_nan_inf_pivot_rules(cuda, lookahead):
    """Special values follow the reference's strict '>' scan (_jit.py:163-170): a NaN candidate is never
    taken unless it is on the diagonal, +-inf wins, ties go to the smallest row."""
    import warnings

    rng = np.random.default_rng(31)
    a = rng.uniform(-1.0, 1.0, (300, 300))
    a[17, 3] = np.nan          # below the diagonal of column 3: must not be chosen
    a[5, 5] = np.nan           # a NaN diagonal candidate
    a[200, 40] = np.inf        # must win column 40 (if still finite there)
    a[100, 60] = -np.inf
    a[150, 80] = a[151, 80] = 7.0   # exact tie: smaller row wins
    ref, rpiv, rinfo = oracle.getrf(a, 64)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        for exact in (True, False):
            lu, piv, info = run(a, 64, lookahead, exact=exact)
            assert np.array_equal(piv, rpiv), exact
            assert info == rinfo
            if exact:
                assert np.array_equal(lu, ref, equal_nan=True)


@pytest.mark.parametrize("env", [{"PFLU_TUR_SPLIT": "1"}, {"PFLU_TUR_SPLIT": "0"}])
def test_schedule_variants_child(cuda, env):
    """The look-ahead schedules selected when libpflu loads (split-overlap vs column-chunk dataflow)
    in a child process: exact mode bitwise = the reference (C1 sha, a ragged case), DMMA mode the
    reference's pivots at C1 and C2."""
    import subprocess
    import sys

    code = (
        "import sys, json, hashlib, numpy as np; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')\n"
        "import oracle; from paper_1804_07017_b200 import lu_factor\n"
        "cf = json.load(open('tests/golden/configs.json')); pv = np.load('tests/golden/configs_pivots.npz')\n"
        "a = np.random.default_rng(0).uniform(-1.0, 1.0, size=(2048, 2048))\n"
        "lu, piv = lu_factor(a.copy(), b=128, lookahead=1, exact=True)\n"
        "assert hashlib.sha256(lu.tobytes()).hexdigest() == cf['c1']['sha256_factors']\n"
        "lu2, piv2 = lu_factor(a.copy(), b=128, lookahead=1)\n"
        "assert np.array_equal(piv2, pv['c1']) and oracle.max_rel_diff(lu2, lu, a) <= 1e-8\n"
        "r = np.random.default_rng(11).uniform(-1, 1, (1000, 1000)); ref, rp, _ = oracle.getrf(r, 96)\n"
        "lu3, p3 = lu_factor(r.copy(), b=96, lookahead=1, exact=True)\n"
        "assert lu3.tobytes() == ref.tobytes() and np.array_equal(p3, rp)\n"
        "c2 = np.random.default_rng(1).uniform(-1.0, 1.0, size=(8192, 8192))\n"
        "lu4, p4 = lu_factor(c2, b=256, lookahead=1)\n"
        "assert np.array_equal(p4, pv['c2'])\n"
        "print('schedule ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, **env), capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "schedule ok" in out.stdout, out.stderr[-3000:]


@pytest.mark.parametrize("lookahead", [0, 1])
def test_trace_hook(cuda, lookahead):
    """The reference's trace semantics (factor.py:104-122, test_factor.py:423-441): a PF record for every
    step, TU (depth 0) or TU_L/TU_R (depth 1) records, ordered timestamps; the GEMM records carry the
    trailing update's algorithmic flops."""
    import torch
    from paper_1804_07017_b200 import getrf_device

    n, b = 1000, 128
    a = torch.from_numpy(np.random.default_rng(21).uniform(-1, 1, (n, n))).cuda()
    tr = []
    piv, info = getrf_device(a, b, lookahead, trace=tr)
    steps = -(-n // b)
    assert info == 0
    pf = sorted(e.k for e in tr if e.label == "PF")
    assert pf == list(range(steps))
    for e in tr:
        assert 0.0 <= e.start <= e.end
    pf_ev = {e.k: e for e in tr if e.label == "PF"}
    for k in range(1, steps):
        assert pf_ev[k].start >= pf_ev[k - 1].end - 1e-6      # panels are a chain
    gemm = sum(e.flop for e in tr if e.label == "GEMM")
    if lookahead == 0:
        assert sorted(e.k for e in tr if e.label == "TU") == list(range(steps - 1))  # the last has no trailing columns
        want = sum(2.0 * (n - (k + 1) * b) ** 2 * b for k in range(steps) if (k + 1) * b < n)
    else:
        assert sorted(e.k for e in tr if e.label == "TU_L") == list(range(steps - 1))
        assert {e.k for e in tr if e.label == "TU_R"} <= set(range(steps))
        want = sum(2.0 * (n - (k + 1) * b) * (n - (k + 2) * b) * b for k in range(steps) if (k + 2) * b < n)
    assert gemm == pytest.approx(want, rel=1e-12)


def test_multipliers_bounded(cuda):
    """Partial pivoting keeps every multiplier |l| <= 1 (+ rounding), test_factor.py:48-53 / 391-398 --
    in the DMMA path too."""
    a0 = config_matrix("c1")
    lu, piv, _ = run(a0, 128, 1, exact=False)
    low = np.tril(lu, -1)
    assert np.max(np.abs(low)) <= 1.0 + 4 * oracle.UNIT_ROUNDOFF


@pytest.mark.parametrize("mode", [1, 2], ids=["la_static", "la_mb"])
@pytest.mark.parametrize("n,b", [(777, 100), (2048, 128), (5000, 256), (8192, 256)])
def test_malleable_schedules_bitwise_equal_dynamic(cuda, mode, n, b):
    """The SM-partitioned look-ahead (persistent trailing GEMM over an atomic tile queue, the panel's
    SMs reserved; LA_MB adds the join grid) computes every tile with the same instructions as the
    dynamic tile-per-CTA schedule: factors and pivots BITWISE equal, pivots = the oracle's."""
    import torch

    from paper_1804_07017_b200 import getrf_device

    a0 = np.random.default_rng(n + b).uniform(-1.0, 1.0, (n, n))
    d0 = torch.from_numpy(a0).to(cuda)
    ref = d0.clone()
    piv_r, info_r = getrf_device(ref, b, 1)
    for rep in range(2):
        x = d0.clone()
        piv, info = getrf_device(x, b, 1, malleable=mode)
        torch.cuda.synchronize()
        assert info == info_r == 0
        assert torch.equal(piv, piv_r)
        assert bitwise_equal(x.cpu().numpy(), ref.cpu().numpy())
    if n <= 2048:
        _, wpiv, _ = oracle.getrf(a0, b)
        assert np.array_equal(piv_r.cpu().numpy(), wpiv)


def test_dmf_la_malleable_runs_la_mb(cuda, golden_small):
    """dmf_la(malleable=True) -> Strategy.LA_MB on the partitioned + join schedule, same result."""
    from paper_1804_07017_b200 import CacheConfig, Kind, Matrix, dmf_la

    a0 = golden_small["u300__a"]
    out = dmf_la(Matrix.from_array(a0.copy()), CacheConfig(b=32), None, Kind.LU, malleable=True)
    assert out.strategy.name == "LA_MB"
    assert np.array_equal(np.asarray(out.pivots) - 1, golden_small["u300__piv"])
    assert oracle.max_rel_diff(np.ascontiguousarray(out.matrix.array), golden_small["u300__f"], a0) <= 1e-10


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_integer_matrices_exact_ties(cuda, seed):
    """Small-integer matrices: many candidates tie EXACTLY in the pivot search (the strict '>' scan of
    _jit.py:163-170 takes the smallest row).  Exact mode must be bitwise the oracle; DMMA mode's pivots
    must equal the oracle's or first differ at a column whose top-two candidates tie within 1e-12 with
    the runner-up taken (north_star's tie rule, classified from the instrumented oracle's record)."""
    from paper_1804_07017_b200 import lu_factor

    rng = np.random.default_rng(100 + seed)
    n, b = 300, 32
    a0 = rng.integers(-2, 3, (n, n)).astype(np.float64)
    a0 += np.eye(n) * 0.5          # keep it nonsingular-ish; ties stay exact in early columns
    want, wpiv, winfo = oracle.getrf(a0, b)
    w = np.array(a0, copy=True)
    piv_t, top2, _ = oracle.getrf_top2_inplace(w, b)
    assert np.array_equal(piv_t, wpiv) and w.tobytes() == want.tobytes()
    ties = oracle.near_ties(top2, 1e-6)
    assert len(ties) > 0                         # the case really has (near-)ties
    for la in (0, 1):
        lu, piv, info = lu_factor(a0.copy(), b=b, lookahead=la, exact=True, return_info=True)
        assert info == winfo and np.array_equal(piv, wpiv) and bitwise_equal(lu, want)
        lu2, piv2 = lu_factor(a0.copy(), b=b, lookahead=la)
        verdict = oracle.classify_pivots(piv2, wpiv, ties)
        assert verdict["ok"], verdict
        if verdict["equal"]:
            assert oracle.max_rel_diff(lu2, want, a0) <= 1e-8
        assert oracle.lu_residual(a0, lu2, piv2) <= 10
