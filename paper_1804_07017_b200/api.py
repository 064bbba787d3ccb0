"""Drop-in LU entry points for the reference package `panelforge` (arXiv 1804.07017).

Primary entry (north_star): :func:`lu_factor` -- float64 n x n in, block size ``b`` and
look-ahead depth in; packed L\\U factors and a 0-based pivot vector out.

Reference-compatible surface (pkg/src/panelforge/factor.py): :func:`dmf_la` (static
look-ahead, factor.py:455-515), :func:`dmf_mtb` (fork-join, factor.py:382-412), :class:`LuOutput`
(factor.py:51-62), :class:`Kind`, :class:`Strategy`, :func:`flops` (factor.py:208-215),
:class:`CacheConfig` and :class:`Matrix` (core.py:17-112).  Every factorization runs on the
B200 through libpflu.so (include/pflu.h); there is no CPU path.
"""
from __future__ import annotations

import ctypes
import enum
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib


class Kind(enum.Enum):
    LU = "lu"
    QR = "qr"


class Strategy(enum.Enum):
    MTB = "mtb"
    RTM = "rtm"
    LA = "la"
    LA_MB = "la-mb"


@dataclass(frozen=True)
class CacheConfig:
    """Blocking parameters (reference core.py:17-52).  Only ``b`` (the panel width) affects the
    GPU factorization; the CPU cache-tiling fields are accepted for signature compatibility."""

    mc: int = 72
    nc: int = 4032
    kc: int = 256
    mr: int = 8
    nr: int = 6
    b: int = 192

    def __post_init__(self):
        for name in ("mc", "nc", "kc", "mr", "nr", "b"):
            if getattr(self, name) < 1:
                raise ValueError(f"CacheConfig.{name} must be >= 1")


class Matrix:
    """Column-major float64 matrix, the reference's container (core.py:55-112): element (i, j)
    at flat offset i + j*leading_dim of a Fortran-ordered (leading_dim, cols) ndarray."""

    __slots__ = ("rows", "cols", "leading_dim", "data")

    def __init__(self, rows: int, cols: int, data: np.ndarray | None = None, leading_dim: int | None = None):
        ld = rows if leading_dim is None else leading_dim
        if ld < rows:
            raise ValueError("leading_dim must be >= rows")
        if data is None:
            data = np.zeros((ld, cols), dtype=np.float64, order="F")
        if data.shape != (ld, cols):
            raise ValueError(f"backing array must have shape ({ld}, {cols})")
        if data.dtype != np.float64 or not data.flags.f_contiguous:
            raise ValueError("backing array must be float64 and column-major")
        self.rows, self.cols, self.leading_dim, self.data = rows, cols, ld, data

    @classmethod
    def zeros(cls, rows: int, cols: int) -> "Matrix":
        return cls(rows, cols)

    @classmethod
    def from_array(cls, arr) -> "Matrix":
        a = np.asfortranarray(np.asarray(arr, dtype=np.float64))
        if a.ndim != 2:
            raise ValueError("expected a 2-D array")
        return cls(a.shape[0], a.shape[1], data=a)

    @classmethod
    def random_uniform(cls, rows: int, cols: int, seed: int) -> "Matrix":
        return cls.from_array(np.random.default_rng(seed).random((rows, cols)))

    @property
    def array(self) -> np.ndarray:
        return self.data[: self.rows, :]

    def copy(self) -> "Matrix":
        return Matrix(self.rows, self.cols, data=self.data.copy(order="F"), leading_dim=self.leading_dim)

    def __repr__(self):
        return f"Matrix({self.rows}x{self.cols}, ld={self.leading_dim})"


@dataclass
class LuOutput:
    """In-place LU factors plus 1-based pivots of length min(m, n) (reference factor.py:51-62).
    ``info`` is 0 or the 1-based first column whose pivot was exactly zero."""

    matrix: Matrix
    pivots: np.ndarray
    strategy: Strategy
    info: int = 0


@dataclass
class QrOutput:
    """In-place QR factors: R in the upper triangle, Householder vectors (unit head, stored below
    the diagonal) and their tau scalars (reference factor.py:65-72)."""

    matrix: Matrix
    tau: np.ndarray
    strategy: Strategy


@dataclass(frozen=True)
class TraceEvent:
    """One timed task (reference factor.py:104-113); times are seconds from the start."""

    label: str
    k: int
    j: int | None
    start: float
    end: float
    worker: int | None
    flop: float = 0.0   # algorithmic flops of the traced work (GEMM records)


def flops(kind: Kind, n: int) -> int:
    """2n^3/3 for LU, 4n^3/3 for QR, rounded to nearest (reference factor.py:208-215)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    num = (2 if kind is Kind.LU else 4) * n ** 3
    q, r = divmod(num, 3)
    return q + (1 if 2 * r >= 3 else 0)


def _validate_shape(m: int, n: int):
    # reference factor.py:293-297
    if m < n:
        raise ValueError("factorizations require a square or tall matrix")
    if n < 1:
        raise ValueError("matrix must be non-empty")


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def getrf_host(a: np.ndarray, b: int, lookahead: int, exact: bool = False, panel_ctas: int = 0,
               panel_kernel: int = 0, malleable: int = 0):
    """Factor a row-major C-contiguous float64 host array in place through pflu_getrf.
    ``malleable``: the look-ahead-1 trailing-update schedule (pflu_options.malleable: 0 dynamic tiles,
    1 SM-partitioned LA, 2 LA_MB = partition + join grid).  Returns (piv0 int64[n], info)."""
    L = _lib.load()
    m, n = a.shape
    piv = np.empty(n, dtype=np.int64)
    info = ctypes.c_int64(0)
    opt = _lib.options(exact=exact, panel_ctas=panel_ctas, panel_kernel=panel_kernel, malleable=malleable)
    rc = L.pflu_getrf(a.ctypes.data, m, n, a.strides[0] // 8, int(b), int(lookahead), piv.ctypes.data,
                      ctypes.byref(info), ctypes.byref(opt))
    _lib.check(rc, "pflu_getrf")
    return piv, int(info.value)


def getrf_device(a, b: int, lookahead: int, exact: bool = False, panel_ctas: int = 0, piv=None, trace=None,
                 panel_kernel: int = 0, malleable: int = 0):
    """Factor a row-major CUDA float64 torch tensor in place through pflu_getrf_device on the
    current torch stream.  Returns (piv0 int64 CUDA tensor, info).  If ``trace`` is a list, it
    receives :class:`TraceEvent` records (labels PF / TU / TU_L / TU_R / GEMM, seconds from the
    start, CUDA-event timed) -- the reference's trace hook (factor.py:104-122)."""
    import torch

    L = _lib.load()
    m, n = a.shape
    if piv is None:
        piv = torch.empty(n, dtype=torch.int64, device=a.device)
    info = ctypes.c_int64(0)
    opt = _lib.options(exact=exact, panel_ctas=panel_ctas, panel_kernel=panel_kernel, malleable=malleable)
    stream = torch.cuda.current_stream(a.device).cuda_stream
    tbuf, tcap, tlen = None, 0, ctypes.c_int(0)
    if trace is not None:
        steps = -(-n // max(1, min(b, n)))
        tcap = 24 * steps + 32
        tbuf = (_lib.TraceEvent * tcap)()
    with torch.cuda.device(a.device):
        rc = L.pflu_getrf_device(a.data_ptr(), m, n, a.stride(0), int(b), int(lookahead), piv.data_ptr(),
                                 ctypes.byref(info), stream, ctypes.byref(opt), tbuf, tcap, ctypes.byref(tlen))
    _lib.check(rc, "pflu_getrf_device")
    if trace is not None:
        for i in range(tlen.value):
            e = tbuf[i]
            lab = _lib.TRACE_LABELS.get(e.label, str(e.label))
            j = e.k + 1 if lab == "TU_L" else None
            trace.append(TraceEvent(lab, int(e.k), j, e.start_ms * 1e-3, e.end_ms * 1e-3, None, float(e.flop)))
    return piv, int(info.value)


def init_gpus(n_gpus: int, devices=None) -> None:
    """pflu_init: hold a multi-GPU context (NCCL communicators, per-rank streams and workspaces) for
    ``n_gpus`` ranks on ``devices`` (default 0 .. n_gpus-1; a repeated device makes ranks share it
    and exchange by copies -- the single-GPU test setup)."""
    L = _lib.load()
    devs = list(range(n_gpus)) if devices is None else [int(d) for d in devices]
    if len(devs) != n_gpus:
        raise ValueError("devices must list one device per rank")
    arr = (ctypes.c_int * n_gpus)(*devs)
    _lib.check(L.pflu_init(int(n_gpus), arr), "pflu_init")


def finalize_gpus() -> None:
    """pflu_finalize: destroy the multi-GPU context."""
    _lib.check(_lib.load().pflu_finalize(), "pflu_finalize")


def getrf_mg(a: np.ndarray, b: int, lookahead: int, n_gpus: int, exact: bool = False, trace=None):
    """pflu_getrf_mg on a square row-major float64 HOST array (in place).  Returns (piv, info);
    ``trace`` (a list) receives rank 0's PF / TU_L / TU_R / TU / BCAST records."""
    L = _lib.load()
    n = a.shape[0]
    if a.ndim != 2 or a.shape[1] != n or a.dtype != np.float64 or not a.flags.c_contiguous:
        raise ValueError("the multi-GPU path factors square row-major float64 matrices")
    piv = np.empty(n, dtype=np.int64)
    info = ctypes.c_int64(0)
    opt = _lib.options(exact=exact)
    tbuf, tcap, tlen = None, 0, ctypes.c_int(0)
    if trace is not None:
        tcap = 8 * (-(-n // max(1, min(b, n)))) + 32
        tbuf = (_lib.TraceEvent * tcap)()
    rc = L.pflu_getrf_mg(a.ctypes.data, n, a.strides[0] // 8, int(b), int(lookahead), int(n_gpus),
                         piv.ctypes.data, ctypes.byref(info), ctypes.byref(opt), tbuf, tcap, ctypes.byref(tlen))
    _lib.check(rc, "pflu_getrf_mg")
    if trace is not None:
        for i in range(tlen.value):
            e = tbuf[i]
            lab = _lib.TRACE_LABELS.get(e.label, str(e.label))
            trace.append(TraceEvent(lab, int(e.k), e.k + 1 if lab == "TU_L" else None, e.start_ms * 1e-3,
                                    e.end_ms * 1e-3, None, float(e.flop)))
    return piv, int(info.value)


def _lu_factor_mg(a, b, lookahead, n_gpus, exact, return_info, overwrite_a):
    arr = np.asarray(a.cpu().numpy() if _is_torch(a) else a)
    if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
        raise ValueError("the multi-GPU path factors square matrices")
    if overwrite_a and arr is a and arr.dtype == np.float64 and arr.flags.c_contiguous and arr.flags.writeable:
        work = arr
    else:
        work = np.array(arr, dtype=np.float64, order="C", copy=True)
    piv, info = getrf_mg(work, b, lookahead, n_gpus, exact=exact)
    if info:
        warnings.warn(f"exactly singular: zero pivot in column {info} (1-based)", RuntimeWarning, stacklevel=3)
    return (work, piv, info) if return_info else (work, piv)


def lu_factor(a, b: int = 256, lookahead: int = 1, n_gpus: int = 1, overwrite_a: bool = True,
              exact: bool = False, return_info: bool = False, panel_ctas: int = 0, panel_kernel: int = 0,
              malleable: int = 0):
    """Blocked right-looking LU with partial pivoting on the B200.

    ``a``: float64 m x n (m >= n) row-major -- a numpy array (host buffers: staged through
    pflu_getrf) or a CUDA torch tensor (device buffers, current stream).  ``lookahead`` 1 is the
    reference's dmf_la, 0 its dmf_mtb.  ``exact=True`` reproduces the reference's rounding in
    every update (bitwise-equal factors); the default runs the trailing update on DMMA tensor
    cores.  ``n_gpus > 1`` runs the 1-D block-cyclic multi-GPU driver: inside an initialised
    torch.distributed group of several processes (one rank per GPU) the torch.distributed driver,
    otherwise -- one process, as the reference's in-process call -- pflu_getrf_mg over n_gpus
    devices (NCCL broadcast per step).  ``panel_kernel`` forces the
    panel factorization of every step (0 automatic, 1 cooperative grid, 2 cluster, 3 recursive).
    ``malleable`` selects the look-ahead-1 trailing-update schedule: 0 dynamic (one CTA per GEMM
    tile; the block scheduler hands the panel's SMs back as soon as it exits), 1 SM-partitioned (the
    reference's LA: the panel's SMs stay with the panel chain), 2 LA_MB (partitioned, plus a join
    grid that puts the panel's SMs on the remaining tiles after PF(k+1)).  All three give bitwise
    identical factors.

    Returns ``(lu, piv)`` (``(lu, piv, info)`` with ``return_info``): packed unit-lower L below
    the diagonal and U on/above it, and 0-based LAPACK pivots (row i swapped with piv[i]).
    """
    if lookahead not in (0, 1):
        raise ValueError("lookahead must be 0 or 1 (the reference defines depth 0 and 1)")
    if b < 1:
        raise ValueError("block size must be >= 1")
    if n_gpus > 1:
        import torch.distributed as tdist

        if tdist.is_available() and tdist.is_initialized() and tdist.get_world_size() > 1:
            # one process per GPU (torchrun): the torch.distributed driver
            from .dist import lu_factor_dist

            return lu_factor_dist(a, b=b, lookahead=lookahead, exact=exact, return_info=return_info)
        # one process, n_gpus devices: the C ABI's multi-GPU driver (pflu_getrf_mg, NCCL)
        return _lu_factor_mg(a, b, lookahead, n_gpus, exact, return_info, overwrite_a)
    if _is_torch(a):
        import torch

        if a.dtype != torch.float64 or a.dim() != 2:
            raise ValueError("expected a 2-D float64 tensor")
        _validate_shape(*a.shape)
        if not a.is_cuda:
            raise ValueError("torch input must be a CUDA tensor (use a numpy array for host buffers)")
        work = a if (overwrite_a and a.stride(1) == 1) else a.contiguous().clone()
        piv, info = getrf_device(work, b, lookahead, exact=exact, panel_ctas=panel_ctas, panel_kernel=panel_kernel,
                                 malleable=malleable)
    else:
        arr = np.asarray(a)
        if arr.dtype != np.float64 or arr.ndim != 2:
            arr = np.asarray(arr, dtype=np.float64)
            if arr.ndim != 2:
                raise ValueError("expected a 2-D array")
        _validate_shape(*arr.shape)
        if overwrite_a and arr is a and arr.flags.c_contiguous and arr.flags.writeable:
            work = arr
        else:
            work = np.array(arr, dtype=np.float64, order="C", copy=True)
        piv, info = getrf_host(work, b, lookahead, exact=exact, panel_ctas=panel_ctas, panel_kernel=panel_kernel,
                               malleable=malleable)
    if info:
        warnings.warn(f"exactly singular: zero pivot in column {info} (1-based)", RuntimeWarning, stacklevel=2)
    return (work, piv, info) if return_info else (work, piv)


def geqrf_host(a: np.ndarray, b: int, lookahead: int) -> np.ndarray:
    """Householder QR of a row-major C-contiguous float64 host array in place through pflu_geqrf.
    Returns tau float64[n]."""
    L = _lib.load()
    m, n = a.shape
    tau = np.zeros(n)
    rc = L.pflu_geqrf(a.ctypes.data, m, n, a.strides[0] // 8, int(b), int(lookahead), tau.ctypes.data)
    _lib.check(rc, "pflu_geqrf")
    return tau


def geqrf_device(a, b: int, lookahead: int, tau=None, trace=None):
    """Householder QR of a row-major CUDA float64 torch tensor in place through pflu_geqrf_device
    on the current torch stream.  Returns tau (float64 CUDA tensor of length n).  ``trace``: as for
    :func:`getrf_device` (PF / TU or PF / TU_L / TU_R records)."""
    import torch

    L = _lib.load()
    m, n = a.shape
    if tau is None:
        tau = torch.zeros(n, dtype=torch.float64, device=a.device)
    stream = torch.cuda.current_stream(a.device).cuda_stream
    tbuf, tcap, tlen = None, 0, ctypes.c_int(0)
    if trace is not None:
        steps = -(-n // max(1, min(b, n)))
        tcap = 8 * steps + 32
        tbuf = (_lib.TraceEvent * tcap)()
    with torch.cuda.device(a.device):
        rc = L.pflu_geqrf_device(a.data_ptr(), m, n, a.stride(0), int(b), int(lookahead), tau.data_ptr(), stream,
                                 tbuf, tcap, ctypes.byref(tlen))
    _lib.check(rc, "pflu_geqrf_device")
    if trace is not None:
        for i in range(tlen.value):
            e = tbuf[i]
            lab = _lib.TRACE_LABELS.get(e.label, str(e.label))
            j = e.k + 1 if lab == "TU_L" else None
            trace.append(TraceEvent(lab, int(e.k), j, e.start_ms * 1e-3, e.end_ms * 1e-3, None, float(e.flop)))
    return tau


def qr_factor(a, b: int = 256, lookahead: int = 1, overwrite_a: bool = True, n_gpus: int = 1):
    """Blocked Householder QR on the B200 (the reference's Kind.QR of dmf_la / dmf_mtb).

    ``a``: float64 m x n (m >= n) row-major -- a numpy array (host buffers, pflu_geqrf) or a CUDA
    torch tensor (device buffers, current stream).  Returns ``(f, tau)``: R on and above the
    diagonal of ``f``, the Householder vectors' tails below it (unit heads implicit), and the
    reflector scalars (H_j = I - tau_j v_j v_j^T, Q = H_1 ... H_n).  ``n_gpus > 1`` runs the 1-D
    block-cyclic multi-GPU driver (dist.geqrf_block_cyclic; an initialised torch.distributed group
    with one rank per GPU); every rank gets the full factors.
    """
    if lookahead not in (0, 1):
        raise ValueError("lookahead must be 0 or 1 (the reference defines depth 0 and 1)")
    if b < 1:
        raise ValueError("block size must be >= 1")
    if n_gpus > 1:
        from .dist import qr_factor_dist

        return qr_factor_dist(a, b=b, lookahead=lookahead)
    if _is_torch(a):
        import torch

        if a.dtype != torch.float64 or a.dim() != 2:
            raise ValueError("expected a 2-D float64 tensor")
        _validate_shape(*a.shape)
        if not a.is_cuda:
            raise ValueError("torch input must be a CUDA tensor (use a numpy array for host buffers)")
        work = a if (overwrite_a and a.stride(1) == 1) else a.contiguous().clone()
        return work, geqrf_device(work, b, lookahead)
    arr = np.asarray(a)
    if arr.dtype != np.float64 or arr.ndim != 2:
        arr = np.asarray(arr, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError("expected a 2-D array")
    _validate_shape(*arr.shape)
    if overwrite_a and arr is a and arr.flags.c_contiguous and arr.flags.writeable:
        work = arr
    else:
        work = np.array(arr, dtype=np.float64, order="C", copy=True)
    return work, geqrf_host(work, b, lookahead)


def _factor_matrix(a, cfg: CacheConfig, kind: Kind, lookahead: int, strategy: Strategy, trace,
                   malleable: int = 0):
    if isinstance(a, Matrix):
        mat = a
    else:
        mat = Matrix.from_array(a)
    _validate_shape(mat.rows, mat.cols)
    # the GPU works row-major; the reference container is column-major -> stage through a
    # row-major copy and write the factors back into the caller's buffer (in place, like the
    # reference, factor.py:300-302)
    work = np.ascontiguousarray(mat.array)
    if trace is not None:
        # the reference's trace hook (factor.py:104-122): run through the device-buffer entry point,
        # which records CUDA-event timed PF / TU / TU_L / TU_R tasks into ``trace``
        import torch

        dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
        if dev is None:
            raise RuntimeError("libpflu needs a CUDA device (there is no CPU fallback)")
        t = torch.from_numpy(work).to(dev)
        if kind is Kind.QR:
            tau = geqrf_device(t, cfg.b, lookahead, trace=trace).cpu().numpy()
            mat.array[...] = t.cpu().numpy()
            return QrOutput(mat, tau, strategy)
        piv, info = getrf_device(t, cfg.b, lookahead, trace=trace, malleable=malleable)
        mat.array[...] = t.cpu().numpy()
        return LuOutput(mat, piv.cpu().numpy() + 1, strategy, info)
    if kind is Kind.QR:
        tau = geqrf_host(work, cfg.b, lookahead)
        mat.array[...] = work
        return QrOutput(mat, tau, strategy)
    piv0, info = getrf_host(work, cfg.b, lookahead, malleable=malleable)
    mat.array[...] = work
    return LuOutput(mat, piv0 + 1, strategy, info)


def dmf_la(a, cfg: CacheConfig, pool=None, kind: Kind = Kind.LU, malleable: bool = False, trace=None):
    """Static look-ahead driver (depth 1), reference factor.py:455-515.  ``pool`` is accepted
    for signature compatibility (the two sections run as two CUDA streams).  ``malleable=True``
    (LA_MB) runs the SM-partitioned trailing update with the join grid (the panel's SMs rejoin the
    GEMM's tile queue after PF(k+1), runtime.py:99-113); ``False`` the dynamic tile schedule."""
    return _factor_matrix(a, cfg, kind, 1, Strategy.LA_MB if malleable else Strategy.LA, trace,
                          malleable=_lib.SCHED_LA_MB if malleable else _lib.SCHED_DYNAMIC)


def dmf_mtb(a, cfg: CacheConfig, pool=None, kind: Kind = Kind.LU, trace=None):
    """Fork-join driver (depth 0), reference factor.py:382-412."""
    return _factor_matrix(a, cfg, kind, 0, Strategy.MTB, trace)
