"""CPU oracle for the LU hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference)
may import this package, and only as the checker / CPU baseline -- never as the thing
measured or shipped.  The product package (paper_1804_07017_b200) never imports it.

`pflu_oracle.c` restates the reference's arithmetic op for op (see its header for the
file:line map into pkg/src/panelforge/).  It is pinned bit-for-bit against vectors that the
reference itself produced (tests/golden/, made by tests/golden/make_golden.py) by
tests/test_oracle.py.  The numpy helpers below restate the reference's residual definition
(pkg/src/panelforge/oracle.py:18, 58-89).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

#: 64-bit unit roundoff used by every normalized residual (reference oracle.py:18).
UNIT_ROUNDOFF = 2.0 ** -53

_d = ctypes.POINTER(ctypes.c_double)
_i = ctypes.POINTER(ctypes.c_int64)
_I64 = ctypes.c_int64


def build() -> str:
    path = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "pflu_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return path


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.orc_lu_unb.restype = _I64
        L.orc_lu_unb.argtypes = [_d, _I64, _I64, _I64, _i, _I64]
        L.orc_laswp.restype = None
        L.orc_laswp.argtypes = [_d, _I64, _I64, _I64, _i, _I64, _I64]
        L.orc_trsm_llnu.restype = None
        L.orc_trsm_llnu.argtypes = [_d, _I64, _I64, _d, _I64, _I64]
        L.orc_gemm_sub.restype = None
        L.orc_gemm_sub.argtypes = [_d, _I64, _d, _I64, _d, _I64, _I64, _I64, _I64]
        L.orc_getrf.restype = _I64
        L.orc_getrf.argtypes = [_d, _I64, _I64, _I64, _I64, _i]
        L.orc_getrf_steps.restype = _I64
        L.orc_getrf_steps.argtypes = [_d, _I64, _I64, _I64, _I64, _i, _I64]
        L.orc_getrf_steps_top2.restype = _I64
        L.orc_getrf_steps_top2.argtypes = [_d, _I64, _I64, _I64, _I64, _i, _I64, _d]
        L.orc_qr_unb.restype = None
        L.orc_qr_unb.argtypes = [_d, _I64, _I64, _I64, _d]
        L.orc_larft.restype = None
        L.orc_larft.argtypes = [_d, _I64, _I64, _I64, _d, _d]
        L.orc_apply_block_reflector.restype = None
        L.orc_apply_block_reflector.argtypes = [_d, _I64, _I64, _I64, _d, _d, _I64, _I64]
        L.orc_geqrf_steps.restype = None
        L.orc_geqrf_steps.argtypes = [_d, _I64, _I64, _I64, _I64, _d, _I64]
        L.orc_set_threads.restype = None
        L.orc_set_threads.argtypes = [ctypes.c_int]
        _LIB = L
    return _LIB


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


def _dp(a):
    return a.ctypes.data_as(_d)


def _ip(a):
    return a.ctypes.data_as(_i)


def _rowmajor(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or not a.flags.c_contiguous:
        a = np.ascontiguousarray(a)
    return a


def lu_unb(a, steps: int | None = None):
    """In-place unblocked LUpp of a row-major array (reference _jit.py:154-187).
    Returns (piv0 int64[min(m,n) or steps], info)."""
    a = _rowmajor(a)
    m, n = a.shape
    k = min(m, n) if steps is None else min(m, n, steps)
    piv = np.zeros(k, dtype=np.int64)
    info = lib().orc_lu_unb(_dp(a), m, n, n, _ip(piv), -1 if steps is None else steps)
    return a, piv, int(info)


def getrf(a, b: int):
    """Blocked LUpp (reference dmf_mtb/dmf_la, factor.py:382-515) on a COPY of `a`.
    Returns (lu row-major, piv 0-based int64[n], info)."""
    a = np.array(a, dtype=np.float64, order="C", copy=True)
    m, n = a.shape
    if m < n or n < 1:
        raise ValueError("factorizations require a square or tall, non-empty matrix")
    piv = np.zeros(n, dtype=np.int64)
    info = lib().orc_getrf(_dp(a), m, n, n, int(b), _ip(piv))
    return a, piv, int(info)


def getrf_steps_inplace(a: np.ndarray, b: int, nsteps: int, piv: np.ndarray | None = None) -> int:
    """First `nsteps` blocked steps of the reference algorithm, in place on a row-major array
    (the bounded CPU-baseline sample used by bench.py)."""
    m, n = a.shape
    if piv is None:
        piv = np.zeros(n, dtype=np.int64)
    return int(lib().orc_getrf_steps(_dp(a), m, n, a.strides[0] // 8, int(b), _ip(piv), int(nsteps)))


def getrf_top2_inplace(a: np.ndarray, b: int, piv: np.ndarray | None = None):
    """The full blocked factorization in place (row-major, any size that fits in host memory), with
    the tie classifier's record: top2[j] = (|winner|, |runner-up|, runner-up row, number of candidates
    within 1e-12 relative of the winner) of column j's pivot search (reference _jit.py:162-170, strict
    '>' so the smallest row wins).  Returns (piv, top2, info)."""
    m, n = a.shape
    if not a.flags.c_contiguous or a.dtype != np.float64:
        raise ValueError("row-major float64 array required (in place)")
    if piv is None:
        piv = np.zeros(n, dtype=np.int64)
    top2 = np.full((n, 4), -1.0)
    info = int(lib().orc_getrf_steps_top2(_dp(a), m, n, n, int(b), _ip(piv), -1, _dp(top2)))
    return piv, top2, info


#: north_star's tie rule: a pivot may differ only where the top two magnitudes tie within this.
TIE_RTOL = 1e-12


def near_ties(top2: np.ndarray, rtol: float = 1e-6) -> np.ndarray:
    """Rows (col, |winner|, |runner-up|, runner-up row[, tied candidates]) of every column whose
    relative top-two gap (v1 - v2) / v1 is <= rtol (the columns where a correctly rounded factorization
    could pick another pivot).  Committed per config so a GPU pivot mismatch can be classified without
    a host re-run."""
    v1, v2 = top2[:, 0], top2[:, 1]
    with np.errstate(divide="ignore", invalid="ignore"):
        gap = np.where(v1 > 0, (v1 - v2) / v1, np.inf)
    cols = np.nonzero((v2 >= 0) & (gap <= rtol))[0]
    extra = [top2[cols, 3]] if top2.shape[1] > 3 else []
    return np.column_stack([cols.astype(np.float64), v1[cols], v2[cols], top2[cols, 2]] + extra)


def classify_pivots(piv_gpu, piv_ref, ties: np.ndarray, rtol: float = TIE_RTOL) -> dict:
    """North_star's pivot rule: identical, or the FIRST mismatch is a column whose top-two candidate
    magnitudes tie within `rtol` relative and the GPU took the runner-up (everything after a legitimate
    tie break legitimately differs).  `ties` = near_ties(top2) of the reference/oracle run."""
    piv_gpu = np.asarray(piv_gpu, dtype=np.int64)
    piv_ref = np.asarray(piv_ref, dtype=np.int64)
    diff = np.nonzero(piv_gpu != piv_ref)[0]
    if len(diff) == 0:
        return {"equal": True, "first_mismatch": None, "tie": None, "ok": True}
    j = int(diff[0])
    row = ties[ties[:, 0] == j] if len(ties) else ties
    if len(row) == 0:
        return {"equal": False, "first_mismatch": j, "tie": None, "ok": False}
    _, v1, v2, r2 = row[0][:4]
    nties = int(row[0][4]) if len(row[0]) > 4 else 2
    gap = (v1 - v2) / v1
    # a two-way tie must have been broken towards the runner-up; with three or more tied candidates
    # any of them is a legitimate choice (only the runner-up's row is recorded)
    ok = bool(gap <= rtol and (int(r2) == int(piv_gpu[j]) or nties > 2))
    return {"equal": False, "first_mismatch": j, "tie": {"v1": v1, "v2": v2, "rel_gap": gap,
            "runner_up_row": int(r2), "tied_candidates": nties}, "ok": ok}


def step_flops(m: int, n: int, b: int, k: int = 0) -> int:
    """Flops of blocked step k (panel getf2 + trsm + gemm) as the reference executes them."""
    col0 = k * b
    bw = min(b, n - col0)
    mp = m - col0
    f = 0
    for j in range(min(mp, bw)):
        f += (mp - j - 1) + 2 * (mp - j - 1) * (bw - j - 1)
    right = n - col0 - bw
    f += bw * (bw - 1) * right                  # trsm: 2 flops x b(b-1)/2 x cols
    f += 2 * (mp - bw) * right * bw             # gemm
    return f


def lu_prefix(a, steps: int):
    """First `steps` elimination steps on a COPY; rows [0, steps) and piv[:steps] are final."""
    a = np.array(a, dtype=np.float64, order="C", copy=True)
    m, n = a.shape
    piv = np.zeros(min(steps, m, n), dtype=np.int64)
    info = lib().orc_lu_unb(_dp(a), m, n, n, _ip(piv), steps)
    return a, piv, int(info)


def laswp(a, piv0, k1: int, k2: int, c0: int = 0, c1: int | None = None):
    """In place: rows k (k1<=k<k2) swapped with piv0[k], ascending (reference _jit.py:141-151)."""
    a = _rowmajor(a)
    piv = np.ascontiguousarray(piv0, dtype=np.int64)
    lib().orc_laswp(_dp(a), a.shape[1], c0, a.shape[1] if c1 is None else c1, _ip(piv), k1, k2)
    return a


def trsm_llnu(l, x):
    """In place x <- unit_lower(l)^-1 x (reference _jit.py:104-113)."""
    l = _rowmajor(l)
    x = _rowmajor(x)
    lib().orc_trsm_llnu(_dp(l), l.shape[1], l.shape[0], _dp(x), x.shape[1], x.shape[1])
    return x


def gemm_sub(c, a, b):
    """In place c <- c - a @ b, per element p ascending, mul then sub (reference _jit.py:54-80)."""
    c = _rowmajor(c)
    a = _rowmajor(a)
    b = _rowmajor(b)
    m, n = c.shape
    k = a.shape[1]
    lib().orc_gemm_sub(_dp(c), n, _dp(a), a.shape[1], _dp(b), b.shape[1], m, n, k)
    return c


# ---------------------------------------------------------------------------------------
# residuals and parity metrics (restating reference oracle.py:58-89)

def perm_from_pivots(piv0, m: int) -> np.ndarray:
    """Row permutation p with (P A)[i] = A[p[i]] for LAPACK ipiv applied ascending."""
    p = np.arange(m)
    for i, r in enumerate(np.asarray(piv0, dtype=np.int64)):
        if r != i:
            p[i], p[r] = p[r], p[i]
    return p


def lu_residual(a0, lu, piv0, block: int = 2048) -> float:
    """||P A - L U||_F / (n * u * ||A||_F), u = 2^-53 (reference oracle.py:78-89), row-blocked
    so it never materialises more than one block of L U."""
    a0 = np.asarray(a0, dtype=np.float64)
    lu = np.asarray(lu, dtype=np.float64)
    m, n = a0.shape
    kk = min(m, n)
    perm = perm_from_pivots(piv0, m)
    upper = np.triu(lu[:kk, :])
    err2 = 0.0
    for r0 in range(0, m, block):
        r1 = min(m, r0 + block)
        lower = np.tril(lu[r0:r1, :kk], r0 - 1)   # global (i, j) kept iff j < i
        for i in range(r0, min(r1, kk)):
            lower[i - r0, i] = 1.0
        d = a0[perm[r0:r1]] - lower @ upper
        err2 += float(np.sum(d * d))
    norm_a = float(np.linalg.norm(a0))
    err = np.sqrt(err2)
    return err if norm_a == 0.0 else err / (max(n, 1) * UNIT_ROUNDOFF * norm_a)


def max_rel_diff(lu_a, lu_b, a0) -> float:
    """max |LU_a - LU_b| / ||A||_max (north_star's second parity measure)."""
    amax = float(np.max(np.abs(a0)))
    return float(np.max(np.abs(np.asarray(lu_a) - np.asarray(lu_b)))) / (amax if amax else 1.0)


# ---------------------------------------------------------------------------------------
# Householder QR (Kind.QR; reference factor.py:147-205, _jit.py:190-218, oracle.py:90-127)

def qr_unb(a):
    """In place unblocked Householder QR of a row-major m x w panel (m >= w) (reference
    _jit.py:190-218, bitwise).  Returns (a, tau)."""
    a = _rowmajor(a)
    m, w = a.shape
    tau = np.zeros(w)
    lib().orc_qr_unb(_dp(a), m, w, w, _dp(tau))
    return a, tau


def larft(v, tau):
    """T (k x k upper) with I - V T V^T = H_1 ... H_k for the reflectors stored in v
    (reference factor.py:174-189, same loop order; the reference's products use BLAS)."""
    v = _rowmajor(v)
    tau = np.ascontiguousarray(tau, dtype=np.float64)
    m, k = v.shape
    t = np.zeros((k, k))
    lib().orc_larft(_dp(v), m, k, k, _dp(tau), _dp(t))
    return t


def geqrf(a, b: int, nsteps: int = -1):
    """Blocked Householder QR (reference dmf_mtb / dmf_la with Kind.QR) on a COPY of `a`.
    Returns (factors row-major: R on/above the diagonal, reflectors below; tau float64[n])."""
    a = np.array(a, dtype=np.float64, order="C", copy=True)
    m, n = a.shape
    if m < n or n < 1:
        raise ValueError("factorizations require a square or tall, non-empty matrix")
    tau = np.zeros(n)
    lib().orc_geqrf_steps(_dp(a), m, n, n, int(b), _dp(tau), int(nsteps))
    return a, tau


def apply_qt(f, tau, c, block: int = 256):
    """Q^T c for the stored reflectors (f, tau), reflector by reflector in blocks (numpy)."""
    f = np.asarray(f, dtype=np.float64)
    c = np.array(c, dtype=np.float64, copy=True)
    m = f.shape[0]
    for j0 in range(0, len(tau), block):
        j1 = min(len(tau), j0 + block)
        for j in range(j0, j1):
            t = tau[j]
            if t == 0.0:
                continue
            v = np.empty(m - j)
            v[0] = 1.0
            v[1:] = f[j + 1:, j]
            w = v @ c[j:]
            c[j:] -= t * np.outer(v, w)
    return c


def form_q(f, tau) -> np.ndarray:
    """m x m orthogonal factor H_1 ... H_k (reference oracle.py:90-110)."""
    f = np.asarray(f, dtype=np.float64)
    m = f.shape[0]
    q = np.eye(m)
    for j in range(len(tau) - 1, -1, -1):
        t = tau[j]
        if t == 0.0:
            continue
        v = np.zeros(m - j)
        v[0] = 1.0
        v[1:] = f[j + 1:, j]
        w = q[j:, :].T @ v
        q[j:, :] -= t * np.outer(v, w)
    return q


def qr_residual(a0, f, tau):
    """(||A - Q R||_F / (n u ||A||_F), ||Q^T Q - I||_F / (n u)) (reference oracle.py:113-127)."""
    a0 = np.asarray(a0, dtype=np.float64)
    f = np.asarray(f, dtype=np.float64)
    n = max(a0.shape[1], 1)
    q = form_q(f, tau)
    r = np.triu(f)
    norm_a = np.linalg.norm(a0)
    err = np.linalg.norm(a0 - q @ r)
    factor = err / (n * UNIT_ROUNDOFF * norm_a) if norm_a else err
    ortho = np.linalg.norm(q.T @ q - np.eye(q.shape[0])) / (n * UNIT_ROUNDOFF)
    return float(factor), float(ortho)


def qr_backward_error(a0, f, tau) -> float:
    """||Q^T A - R||_F / (n u ||A||_F) without forming Q (large sizes)."""
    a0 = np.asarray(a0, dtype=np.float64)
    n = max(a0.shape[1], 1)
    d = apply_qt(f, tau, a0) - np.triu(np.asarray(f))
    norm_a = np.linalg.norm(a0)
    err = np.linalg.norm(d)
    return float(err / (n * UNIT_ROUNDOFF * norm_a)) if norm_a else float(err)
