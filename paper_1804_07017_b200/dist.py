"""Multi-GPU LU with partial pivoting: 1-D block-cyclic columns + per-step panel broadcast.

SURVEY.md §8(e).  Column block j (width b) lives on rank j % P; every rank stores its blocks
contiguously (row-major n x n_local).  Rows are not distributed, so the row interchanges of
partial pivoting stay local to each rank.  Per step k (owner o = k % P):

  owner o:   PF(k) on its local copy of block k            (pflu_panel, cooperative kernel)
             pack rows [kb, n) of the factored panel         (contiguous (n - kb) x bw buffer)
  all ranks: broadcast panel + pivots from o                 (torch.distributed -> NCCL on GPUs)
             pivot plan; deferred left swaps on local blocks < k
             TU on local blocks > k: laswp + L11^-1 (from the broadcast L11) + DMMA GEMM with L21

Look-ahead (depth 1, dmf_la factor.py:455-515 across ranks): the owner of block k+1 first updates
that block (TU_L) and factors / broadcasts it on a high-priority panel stream while every rank runs
the rest of TU_R(k) on a low-priority update stream; events order TU_R(k+1) after the broadcast of
panel k+1 and TU_L(k+1) after TU_R(k).

The driver is written against a small kernel backend so that the SAME schedule runs
  * on B200s through libpflu.so (CudaKernels: the product path), and
  * on CPU tensors under gloo in tests/test_dist.py, where the test injects a backend built on the
    CPU oracle (tests only; this module never imports the oracle).
"""
from __future__ import annotations

import ctypes
import os

import torch
import torch.distributed as dist

from . import _lib


# ---------------------------------------------------------------------------------------------
# block-cyclic bookkeeping

def num_blocks(n: int, b: int) -> int:
    return -(-n // b)


def local_blocks(n: int, b: int, P: int, r: int) -> list[int]:
    """Global block indices owned by rank r, in local storage order."""
    return list(range(r, num_blocks(n, b), P))


def local_cols(n: int, b: int, P: int, r: int) -> int:
    return sum(min(b, n - j * b) for j in local_blocks(n, b, P, r))


def local_col_of_block(j: int, b: int, P: int) -> int:
    """Local storage column of global block j on its owner (all blocks before the last are full)."""
    return (j // P) * b


def local_cols_before(k: int, n: int, b: int, P: int, r: int) -> int:
    """Number of local columns of rank r that belong to global blocks < k."""
    return sum(min(b, n - j * b) for j in local_blocks(n, b, P, r) if j < k)


def scatter_columns(a_full: torch.Tensor, b: int, P: int, r: int) -> torch.Tensor:
    """Rank r's block-cyclic columns of a full n x n matrix, row-major contiguous."""
    n = a_full.shape[1]
    cols = [a_full[:, j * b: min(n, (j + 1) * b)] for j in local_blocks(n, b, P, r)]
    return torch.cat(cols, dim=1).contiguous() if cols else a_full.new_empty((a_full.shape[0], 0))


def gather_columns(local: list[torch.Tensor], n: int, b: int) -> torch.Tensor:
    """Inverse of scatter_columns given every rank's local block (list indexed by rank)."""
    P = len(local)
    out = local[0].new_empty((local[0].shape[0], n))
    for r in range(P):
        c = 0
        for j in local_blocks(n, b, P, r):
            w = min(b, n - j * b)
            out[:, j * b: j * b + w] = local[r][:, c: c + w]
            c += w
    return out


def allgather_columns(a_loc: torch.Tensor, n: int, b: int, group=None) -> torch.Tensor:
    """All-gather every rank's local columns into the full n x n matrix (padded to equal sizes,
    since ranks own different numbers of columns)."""
    P = dist.get_world_size(group)
    wmax = max(local_cols(n, b, P, q) for q in range(P))
    pad = a_loc.new_zeros((a_loc.shape[0], wmax))
    pad[:, : a_loc.shape[1]] = a_loc
    parts = [torch.empty_like(pad) for _ in range(P)]
    dist.all_gather(parts, pad, group=group)
    return gather_columns([parts[q][:, : local_cols(n, b, P, q)] for q in range(P)], n, b)


# ---------------------------------------------------------------------------------------------
# kernel backend of the product path: libpflu.so on torch CUDA tensors

class CudaKernels:
    """libpflu.so entry points on strided row-major torch CUDA views (pointer + leading dim)."""

    is_cuda = True

    # panels taller than grid_rows run on the cooperative-grid panel kernel (more SMs, lower latency)
    # when the panel chain, not the per-rank trailing update, bounds the run (many ranks); with few
    # ranks the 16-SM cluster kernel leaves more SMs to the update.  None: decided per call from P.
    GRID_PANEL_ROWS = 8192
    GRID_MIN_RANKS = int(os.environ.get("PFLU_DIST_GRID_MIN_RANKS", "4"))  # scaling model: 2 ranks -> cluster; from 4 the (adaptive) multi-cluster kernel

    def __init__(self, device: torch.device, exact: bool = False, grid_rows: int | None = None):
        self.L = _lib.load()
        self.grid_rows = grid_rows
        self.device = device
        self.opt = _lib.options(exact=exact)
        # tall owner panels on the chain-bound rank counts: the multi-cluster kernel (grid kernel where it does not fit)
        self.opt_grid = _lib.options(exact=exact, panel_kernel=int(os.environ.get("PFLU_TALL_KERNEL", _lib.PANEL_MCLUSTER)))
        # the same kernel capped at two clusters (32 SMs): for the steps whose trailing update outlasts the panel
        self.opt_grid2 = _lib.options(exact=exact, panel_ctas=32,
                                      panel_kernel=int(os.environ.get("PFLU_TALL_KERNEL", _lib.PANEL_MCLUSTER)))
        self.ranks = 1  # set by the driver: ranks sharing the trailing update (panel() sizes the tall-panel kernel with it)
        self.exact = exact
        self.fast_solve = not exact  # U12 solve on DMMA with inverted diagonal blocks
        lo, hi = torch.cuda.Stream.priority_range()
        self.sP = torch.cuda.Stream(device=device, priority=hi)
        self.sU = torch.cuda.Stream(device=device, priority=lo)

    # streams / events
    def stream(self, which: str):
        return torch.cuda.stream(self.sP if which == "P" else self.sU)

    def event(self):
        return torch.cuda.Event()

    def record(self, ev, which: str):
        ev.record(self.sP if which == "P" else self.sU)

    def wait(self, ev, which: str):
        (self.sP if which == "P" else self.sU).wait_event(ev)

    def begin(self):
        cur = torch.cuda.current_stream(self.device)
        self.sP.wait_stream(cur)
        self.sU.wait_stream(cur)

    def join(self):
        cur = torch.cuda.current_stream(self.device)
        cur.wait_stream(self.sP)
        cur.wait_stream(self.sU)

    def _st(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    # kernels (asynchronous on the current stream)
    def info_reset(self):
        _lib.check(self.L.pflu_info_reset(self._st()), "pflu_info_reset")

    def info_read(self) -> int:
        v = ctypes.c_int64(0)
        _lib.check(self.L.pflu_info_read(ctypes.byref(v), self._st()), "pflu_info_read")
        return int(v.value)

    def panel(self, a, m: int, d: int, col: int, w: int, piv):
        gr = self.grid_rows if self.grid_rows is not None else self.GRID_PANEL_ROWS
        opt = self.opt_grid if m - d > gr else self.opt
        if opt is self.opt_grid and opt.panel_kernel == _lib.PANEL_MCLUSTER and os.environ.get("PFLU_MC_ADAPT", "1") != "0":
            # = tall_panel_ctas() of csrc/pflu.cu: while this rank's share of the step's trailing update (ms, at
            # the in-step DMMA rate) outlasts the panel + TU_L (measured 0.83 + 1.65e-5 * rows), the step is
            # bound by SM time: two clusters instead of four
            rows = m - d
            t_upd = 2.0 * rows * ((m - d - w) / max(1, self.ranks)) * w / 33.0e12 * 1e3
            if t_upd > 0.83 + 1.65e-5 * rows:
                opt = self.opt_grid2
        rc = self.L.pflu_panel(a.data_ptr(), a.stride(0), m, d, col, w, piv.data_ptr(), None, self._st(),
                               ctypes.byref(opt))
        _lib.check(rc, "pflu_panel")

    def plan(self, piv, d: int, nb: int, plan):
        _lib.check(self.L.pflu_pivot_plan(piv.data_ptr(), d, nb, plan.data_ptr(), self._st()), "pflu_pivot_plan")

    def diag_inv(self, l11, inv):
        _lib.check(self.L.pflu_diag_inv(l11.data_ptr(), l11.stride(0), l11.shape[0], inv.data_ptr(), self._st()),
                   "pflu_diag_inv")

    def swap_trsm(self, a, d: int, nb: int, plan, c0: int, c1: int, l11=None, inv=None):
        if c1 <= c0:
            return
        lp = l11.data_ptr() if l11 is not None else None
        ldl = l11.stride(0) if l11 is not None else nb
        if inv is not None and l11 is not None:
            rc = self.L.pflu_swap_trsm_inv(a.data_ptr(), a.stride(0), d, nb, plan.data_ptr(), c0, c1, lp, ldl,
                                           inv.data_ptr(), self._st())
            _lib.check(rc, "pflu_swap_trsm_inv")
            return
        rc = self.L.pflu_swap_trsm_plan(a.data_ptr(), a.stride(0), d, nb, plan.data_ptr(), c0, c1, lp, ldl,
                                        self._st())
        _lib.check(rc, "pflu_swap_trsm_plan")

    def gemm(self, c, a, b):
        m, n = c.shape
        k = a.shape[1]
        if m == 0 or n == 0 or k == 0:
            return
        rc = self.L.pflu_gemm_update(c.data_ptr(), c.stride(0), a.data_ptr(), a.stride(0), b.data_ptr(),
                                     b.stride(0), m, n, k, int(self.exact), self._st())
        _lib.check(rc, "pflu_gemm_update")

    # Householder QR (Kind.QR)
    def qr_panel(self, a, m: int, d: int, col: int, w: int, tau):
        rc = self.L.pflu_qr_panel(a.data_ptr(), a.stride(0), m, d, col, w, tau.data_ptr(), self._st())
        _lib.check(rc, "pflu_qr_panel")

    def qr_apply(self, v, tau, c):
        mp, k = v.shape
        nc = c.shape[1]
        if nc == 0 or mp == 0:
            return
        rc = self.L.pflu_apply_block_reflector(v.data_ptr(), v.stride(0), mp, k, tau.data_ptr(), c.data_ptr(),
                                               c.stride(0), nc, self._st())
        _lib.check(rc, "pflu_apply_block_reflector")


# ---------------------------------------------------------------------------------------------
# the distributed driver

class _Trace:
    """PF / TU / TU_L / TU_R / BCAST records of one rank (the reference's trace hook, factor.py:104-122;
    SURVEY.md §8(b) adds BCAST): CUDA-event pairs on the stream the work runs on, or host wall
    clock for the CPU test backend."""

    def __init__(self, kernels, out):
        self.k = kernels
        self.out = out
        self.recs = []
        self.cuda = getattr(kernels, "is_cuda", False)
        self.t0 = self._stamp("P")

    def _stamp(self, which):
        if self.cuda:
            e = torch.cuda.Event(enable_timing=True)
            e.record(self.k.sP if which == "P" else self.k.sU)
            return e
        import time

        return time.perf_counter()

    def begin(self, label, k, which):
        return (label, k, which, self._stamp(which))

    def end(self, tok):
        label, k, which, s = tok
        self.recs.append((label, k, s, self._stamp(which)))

    def finish(self):
        from .api import TraceEvent

        if self.cuda:
            torch.cuda.synchronize()
            rel = lambda e: self.t0.elapsed_time(e) * 1e-3  # noqa: E731
        else:
            rel = lambda t: t - self.t0  # noqa: E731
        for label, k, s, e in self.recs:
            self.out.append(TraceEvent(label, k, k + 1 if label == "TU_L" else None, rel(s), rel(e), None, 0.0))


class _NoTrace:
    def begin(self, *a):
        return None

    def end(self, tok):
        pass

    def finish(self):
        pass


def getrf_block_cyclic(a_loc: torch.Tensor, n: int, b: int, lookahead: int = 1, kernels=None, group=None,
                       piv: torch.Tensor | None = None, row_sink=None, trace=None, emulate: int = 0):
    """Factor the block-cyclic distributed n x n matrix in place.

    ``row_sink(r0, r1, events)`` (CUDA only, optional) is called once per step as soon as local rows
    [r0, r1) are final (their trailing update, TU_L and left swaps are enqueued); ``events`` are the
    CUDA events to wait for -- lu_factor_local streams those rows back to the host with it.

    ``a_loc``: this rank's local columns (row-major, n rows, ``local_cols(n, b, P, rank)`` columns).
    Returns ``(piv, info)``: the full 0-based pivot vector (identical on every rank) and the
    1-based first zero-pivot column (0 if none), agreed over all ranks.
    ``trace`` (a list, optional) receives this rank's PF / TU / TU_L / TU_R / BCAST records.
    ``emulate=Q`` (single rank only; the scaling model of tools/emu_scaling.py --driver dist): run the
    critical path of one rank of a Q-rank job with THIS schedule and kernels -- the rank owns and
    factors every panel (as each step's owner would, packing it into the message as for a broadcast)
    but updates only ~1/Q of every trailing matrix and of the left columns; the factors are then not
    a factorization of the input (timing only).
    """
    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    if kernels is None:
        kernels = CudaKernels(a_loc.device)
    if emulate and P != 1:
        raise ValueError("emulate is a single-rank scaling model")
    Q = max(1, int(emulate or 1))  # the rank count whose critical path runs
    if getattr(kernels, "is_cuda", False):
        kernels.ranks = max(P, Q)
    if getattr(kernels, "is_cuda", False) and kernels.grid_rows is None:
        kernels.grid_rows = kernels.GRID_PANEL_ROWS if max(P, Q) >= kernels.GRID_MIN_RANKS else 1 << 62
    dev = a_loc.device
    if a_loc.shape[0] != n or a_loc.shape[1] != local_cols(n, b, P, r) or a_loc.stride(1) != 1:
        raise ValueError("a_loc must be the row-major local block-cyclic columns (n x local_cols)")
    nblk = num_blocks(n, b)
    if piv is None:
        piv = torch.zeros(n, dtype=torch.int64, device=dev)
    # broadcast buffers: the packed panel ((n - kb) x bw) followed by its bw pivots (int64 bits)
    pbuf = [torch.empty(n * b + b, dtype=torch.float64, device=dev) for _ in range(2)]
    plans = [torch.empty(1 + 3 * b, dtype=torch.int64, device=dev) for _ in range(2)]
    fast = getattr(kernels, "fast_solve", False) and b <= 512
    invs = [torch.empty(((b + 31) // 32) * 1024, dtype=torch.float64, device=dev) for _ in range(2)] if fast else [None, None]
    ev_bc = [kernels.event() for _ in range(2)]
    ev_tu = [kernels.event() for _ in range(2)]
    kernels.begin()
    tr = _Trace(kernels, trace) if trace is not None else _NoTrace()
    with kernels.stream("P"):
        kernels.info_reset()

    def cols_before(k):
        return local_cols_before(k, n, b, P, r)

    def pf_pack_bcast(k):
        """Owner: factor block k and pack it; everyone: broadcast + pivot plan (on the panel stream)."""
        col0 = k * b
        bw = min(b, n - col0)
        rows = n - col0
        o = k % P
        msg = pbuf[k % 2][: rows * bw + bw]
        buf = msg[: rows * bw].view(rows, bw)
        pv = msg[rows * bw:].view(torch.int64)
        if r == o:
            lc = local_col_of_block(k, b, P)
            t = tr.begin("PF", k, "P")
            kernels.panel(a_loc, n, col0, lc, bw, piv)
            tr.end(t)
            buf.copy_(a_loc[col0:, lc: lc + bw])
            pv.copy_(piv[col0: col0 + bw])
        if P > 1:
            t = tr.begin("BCAST", k, "P")
            dist.broadcast(msg, src=o, group=group)  # one message per step: panel + pivots
            if r != o:
                piv[col0: col0 + bw].copy_(pv)
            tr.end(t)
        kernels.plan(piv, col0, bw, plans[k % 2])
        if fast:
            kernels.diag_inv(buf[:bw, :bw], invs[k % 2])
        return buf

    def update(k, buf, c0, c1):
        """TU of step k on local columns [c0, c1): laswp + trsm (L11 from the broadcast) + GEMM."""
        if c1 <= c0:
            return
        col0 = k * b
        bw = min(b, n - col0)
        if fast:
            kernels.swap_trsm(a_loc, col0, bw, plans[k % 2], c0, c1, buf[:bw, :bw], invs[k % 2])
        else:
            kernels.swap_trsm(a_loc, col0, bw, plans[k % 2], c0, c1, buf[:bw, :bw])
        if col0 + bw < n:
            kernels.gemm(a_loc[col0 + bw:, c0:c1], buf[bw:, :], a_loc[col0: col0 + bw, c0:c1])

    def share(lo, hi):
        """Emulation: the part of [lo, hi) one of Q ranks updates (~1/Q, block-aligned)."""
        if Q == 1 or hi <= lo:
            return hi
        return min(hi, lo + -(-((hi - lo + Q - 1) // Q) // b) * b)

    def left_swaps(k):
        col0 = k * b
        bw = min(b, n - col0)
        kernels.swap_trsm(a_loc, col0, bw, plans[k % 2], 0, share(0, cols_before(k)), None)

    ncl = a_loc.shape[1]
    if lookahead == 0:
        for k in range(nblk):
            with kernels.stream("P"):
                buf = pf_pack_bcast(k)
                t = tr.begin("TU", k, "P")
                left_swaps(k)
                update(k, buf, cols_before(k + 1), share(cols_before(k + 1), ncl))
                tr.end(t)
                if row_sink is not None:
                    e = kernels.event()
                    kernels.record(e, "P")
                    row_sink(k * b, min(n, (k + 1) * b), [e])
    else:
        bufs = {}
        with kernels.stream("P"):
            bufs[0] = pf_pack_bcast(0)
            kernels.record(ev_bc[0], "P")
        for k in range(nblk):
            nxt = k + 1 < nblk
            # columns of block k+1 on this rank (only its owner has them)
            own_next = nxt and (k + 1) % P == r
            lo_r = cols_before(k + 2) if own_next else cols_before(k + 1)
            with kernels.stream("U"):
                kernels.wait(ev_bc[k % 2], "U")
                t = tr.begin("TU_R", k, "U")
                update(k, bufs[k], lo_r, share(lo_r, ncl))
                left_swaps(k)
                tr.end(t)
                kernels.record(ev_tu[k % 2], "U")
            e_tl = None
            if nxt:
                with kernels.stream("P"):
                    if k > 0:
                        kernels.wait(ev_tu[(k - 1) % 2], "P")
                    if own_next:
                        t = tr.begin("TU_L", k, "P")
                        update(k, bufs[k], cols_before(k + 1), cols_before(k + 2))
                        tr.end(t)
                        if row_sink is not None:
                            e_tl = kernels.event()
                            kernels.record(e_tl, "P")
                    bufs[k + 1] = pf_pack_bcast(k + 1)
                    kernels.record(ev_bc[(k + 1) % 2], "P")
            if row_sink is not None:
                # rows of block row k are final once TU_R(k) + left swaps(k) (U) and TU_L(k) (P) are
                # done: later steps only touch rows below
                e_u = kernels.event()
                kernels.record(e_u, "U")
                row_sink(k * b, min(n, (k + 1) * b), [e_u] + ([e_tl] if e_tl is not None else []))
            bufs.pop(k - 1, None)
    if kernels.is_cuda:
        kernels.join()
    tr.finish()
    with kernels.stream("P"):
        info = kernels.info_read()
    if P > 1:
        t = torch.tensor([info if info > 0 else 2 ** 62], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        info = int(t.item())
        info = 0 if info >= 2 ** 62 else info
    return piv, info


def geqrf_block_cyclic(a_loc: torch.Tensor, n: int, b: int, lookahead: int = 1, kernels=None, group=None,
                       tau: torch.Tensor | None = None):
    """Householder QR (Kind.QR) of the block-cyclic distributed n x n matrix, in place.

    Same distribution and schedule as getrf_block_cyclic: the owner of block k factors it
    (pflu_qr_panel) and broadcasts ONE message -- the (n - kb) x bw panel (R on top, the reflectors
    below) followed by its bw tau -- and every rank applies the block reflector to its local
    trailing columns (pflu_apply_block_reflector, which forms V and T from the message).  Look-ahead
    1: the owner of block k+1 updates it first, factors it and broadcasts it while every rank runs
    the rest of step k's update.  Returns tau (the full n-vector, identical on every rank)."""
    P = dist.get_world_size(group)
    r = dist.get_rank(group)
    if kernels is None:
        kernels = CudaKernels(a_loc.device)
    dev = a_loc.device
    if a_loc.shape[0] != n or a_loc.shape[1] != local_cols(n, b, P, r) or a_loc.stride(1) != 1:
        raise ValueError("a_loc must be the row-major local block-cyclic columns (n x local_cols)")
    nblk = num_blocks(n, b)
    if tau is None:
        tau = torch.zeros(n, dtype=torch.float64, device=dev)
    pbuf = [torch.empty(n * b + b, dtype=torch.float64, device=dev) for _ in range(2)]
    ev_bc = [kernels.event() for _ in range(2)]
    ev_tu = [kernels.event() for _ in range(2)]
    kernels.begin()

    def cols_before(k):
        return local_cols_before(k, n, b, P, r)

    def pf_pack_bcast(k):
        col0 = k * b
        bw = min(b, n - col0)
        rows = n - col0
        o = k % P
        msg = pbuf[k % 2][: rows * bw + bw]
        buf = msg[: rows * bw].view(rows, bw)
        tv = msg[rows * bw:]
        if r == o:
            lc = local_col_of_block(k, b, P)
            kernels.qr_panel(a_loc, n, col0, lc, bw, tau[col0: col0 + bw])
            buf.copy_(a_loc[col0:, lc: lc + bw])
            tv.copy_(tau[col0: col0 + bw])
        if P > 1:
            dist.broadcast(msg, src=o, group=group)  # one message per step: panel + tau
            if r != o:
                tau[col0: col0 + bw].copy_(tv)
        return buf, tv

    def update(k, bt, c0, c1):
        if c1 <= c0:
            return
        buf, tv = bt
        kernels.qr_apply(buf, tv, a_loc[k * b:, c0:c1])

    ncl = a_loc.shape[1]
    if lookahead == 0:
        for k in range(nblk):
            with kernels.stream("P"):
                bt = pf_pack_bcast(k)
                update(k, bt, cols_before(k + 1), ncl)
    else:
        bufs = {}
        with kernels.stream("P"):
            bufs[0] = pf_pack_bcast(0)
            kernels.record(ev_bc[0], "P")
        for k in range(nblk):
            nxt = k + 1 < nblk
            own_next = nxt and (k + 1) % P == r
            lo_r = cols_before(k + 2) if own_next else cols_before(k + 1)
            with kernels.stream("U"):
                kernels.wait(ev_bc[k % 2], "U")
                update(k, bufs[k], lo_r, ncl)
                kernels.record(ev_tu[k % 2], "U")
            if nxt:
                with kernels.stream("P"):
                    if k > 0:
                        kernels.wait(ev_tu[(k - 1) % 2], "P")
                    if own_next:
                        update(k, bufs[k], cols_before(k + 1), cols_before(k + 2))
                    bufs[k + 1] = pf_pack_bcast(k + 1)
                    kernels.record(ev_bc[(k + 1) % 2], "P")
            bufs.pop(k - 1, None)
    if kernels.is_cuda:
        kernels.join()
    return tau


def qr_factor_dist(a, b: int = 256, lookahead: int = 1):
    """``qr_factor(..., n_gpus=P)``: every rank passes the same full n x n matrix; each factors its
    block-cyclic columns on its GPU; every rank gets the full factors (all-gather) and tau."""
    import numpy as np

    if not dist.is_initialized():
        raise RuntimeError("n_gpus > 1 needs an initialised torch.distributed process group (one rank per GPU)")
    P, r = dist.get_world_size(), dist.get_rank()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", r % max(1, torch.cuda.device_count()))))
    torch.cuda.set_device(dev)
    full = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    if full.dim() != 2 or full.shape[0] != full.shape[1] or full.dtype != torch.float64 or full.stride(1) != 1:
        raise ValueError("the multi-GPU path factors square row-major float64 matrices")
    n = full.shape[1]
    a_loc = torch.empty((n, local_cols(n, b, P, r)), dtype=torch.float64, device=dev)
    copy_local_columns(a_loc, full, n, b, P, r, to_device=True)
    tau = geqrf_block_cyclic(a_loc, n, b, lookahead, CudaKernels(dev))
    f = allgather_columns(a_loc, n, b)
    if not isinstance(a, torch.Tensor):
        return f.cpu().numpy(), tau.cpu().numpy()
    return (f if full.is_cuda else f.cpu()), (tau if full.is_cuda else tau.cpu())


def copy_local_columns(dst, src, n: int, b: int, P: int, r: int, to_device: bool, stream=None):
    """Strided copies of rank r's block-cyclic column blocks between a full row-major n x n matrix
    (host, ideally pinned) and the rank's local device buffer (pflu_copy2d per block)."""
    L = _lib.load()
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    nloc = local_cols(n, b, P, r)
    full = src if to_device else dst
    loc = dst if to_device else src
    c = 0
    for j in local_blocks(n, b, P, r):
        w = min(b, n - j * b)
        fptr = full.data_ptr() + j * b * 8
        lptr = loc.data_ptr() + c * 8
        if to_device:
            rc = L.pflu_copy2d(lptr, nloc * 8, fptr, n * 8, w * 8, n, st)
        else:
            rc = L.pflu_copy2d(fptr, n * 8, lptr, nloc * 8, w * 8, n, st)
        _lib.check(rc, "pflu_copy2d")
        c += w


def lu_factor_dist(a, b: int = 256, lookahead: int = 1, exact: bool = False, return_info: bool = False,
                   gather: str = "all"):
    r"""``lu_factor(..., n_gpus=P)``: every rank passes the same full n x n matrix (host numpy / torch,
    or a CUDA tensor); each rank copies only its block-cyclic columns to its GPU and factors them.

    gather="all"   -> every rank gets the full packed L\U (all-gather over NCCL);
    gather="local" -> each rank writes ITS columns of L\U back into ``a`` in place (the distributed
                      result, ScaLAPACK style) -- the cheap path used by bench.py's e2e leg.
    Returns (lu, piv) (+ info): piv is the full 0-based pivot vector on every rank."""
    import numpy as np

    if not dist.is_initialized():
        raise RuntimeError("n_gpus > 1 needs an initialised torch.distributed process group (one rank per GPU)")
    P, r = dist.get_world_size(), dist.get_rank()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", r % max(1, torch.cuda.device_count()))))
    torch.cuda.set_device(dev)
    full = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    if full.dim() != 2 or full.shape[0] != full.shape[1] or full.dtype != torch.float64 or full.stride(1) != 1:
        raise ValueError("the multi-GPU path factors square row-major float64 matrices")
    n = full.shape[1]
    a_loc = torch.empty((n, local_cols(n, b, P, r)), dtype=torch.float64, device=dev)
    copy_local_columns(a_loc, full, n, b, P, r, to_device=True)
    piv, info = getrf_block_cyclic(a_loc, n, b, lookahead, CudaKernels(dev, exact=exact))
    if gather == "local":
        copy_local_columns(full, a_loc, n, b, P, r, to_device=False)
        torch.cuda.synchronize()
        lu = full
    else:
        lu = allgather_columns(a_loc, n, b)
        if not full.is_cuda:
            lu = lu.cpu()
    if not isinstance(a, torch.Tensor):
        lu = lu.numpy() if gather == "all" else a
        piv = piv.cpu().numpy()
    return (lu, piv, info) if return_info else (lu, piv)


def lu_factor_local(a_loc, n: int, b: int = 256, lookahead: int = 1, exact: bool = False,
                    return_info: bool = False):
    r"""Distributed-input form of ``lu_factor(..., n_gpus=P)`` (ScaLAPACK style): each rank passes
    ONLY its block-cyclic columns -- ``a_loc`` of shape (n, local_cols(n, b, P, rank)), row-major,
    host (numpy / torch, ideally pinned) or CUDA -- and gets its columns of the packed L\U back in
    place, plus the full 0-based pivot vector.  Host traffic per rank is 1/P of the matrix."""
    import numpy as np

    if not dist.is_initialized():
        raise RuntimeError("lu_factor_local needs an initialised torch.distributed process group")
    P, r = dist.get_world_size(), dist.get_rank()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", r % max(1, torch.cuda.device_count()))))
    torch.cuda.set_device(dev)
    t = a_loc if isinstance(a_loc, torch.Tensor) else torch.from_numpy(a_loc)
    if t.dim() != 2 or t.shape[0] != n or t.shape[1] != local_cols(n, b, P, r) or t.dtype != torch.float64 \
            or t.stride(1) != 1:
        raise ValueError("a_loc must be this rank's (n x local_cols) row-major float64 block-cyclic columns")
    if t.is_cuda:
        piv, info = getrf_block_cyclic(t, n, b, lookahead, CudaKernels(dev, exact=exact))
        return (t, piv, info) if return_info else (t, piv)
    d = torch.empty(t.shape, dtype=torch.float64, device=dev)
    d.copy_(t, non_blocking=True)
    # every block row streams back to the host as soon as it is final (D2H overlaps the rest)
    cs = torch.cuda.Stream(device=dev)

    def sink(r0, r1, events):
        for e in events:
            cs.wait_event(e)
        with torch.cuda.stream(cs):
            t[r0:r1].copy_(d[r0:r1], non_blocking=True)

    piv, info = getrf_block_cyclic(d, n, b, lookahead, CudaKernels(dev, exact=exact), row_sink=sink)
    piv_h = piv.cpu()
    cs.synchronize()
    torch.cuda.synchronize()
    out_piv = piv_h.numpy() if not isinstance(a_loc, torch.Tensor) else piv_h
    return (a_loc, out_piv, info) if return_info else (a_loc, out_piv)


def local_columns_seeded(n: int, b: int, P: int, r: int, seed: int, dist_name: str = "uniform",
                         chunk_rows: int = 1024, diag_shift: float = 0.0):
    """Rank r's block-cyclic columns of the seeded BASELINE matrix (numpy default_rng(seed), row-major
    draw order), generated in row chunks so no rank ever holds the full n x n matrix."""
    import numpy as np

    g = np.random.default_rng(seed)
    blocks = local_blocks(n, b, P, r)
    out = np.empty((n, local_cols(n, b, P, r)), dtype=np.float64)
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        rows = g.uniform(-1.0, 1.0, size=(r1 - r0, n)) if dist_name == "uniform" else g.standard_normal((r1 - r0, n))
        c = 0
        for j in blocks:
            w = min(b, n - j * b)
            out[r0:r1, c: c + w] = rows[:, j * b: j * b + w]
            c += w
    if diag_shift:
        c = 0
        for j in blocks:
            w = min(b, n - j * b)
            for t in range(w):
                out[j * b + t, c + t] += diag_shift
            c += w
    return out


# ---------------------------------------------------------------------------------------------
# bench.py --gpus N (torchrun, one rank per GPU)

def bench_dist(args, lu_flops, metric, unit, ClockSampler, fp64_peak, configs=None, workload=None):
    import json
    import time

    import numpy as np

    # the communicator log (nranks per communicator) stays on unless the caller chose otherwise
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if not dist.is_initialized():
        for k, v in (("RANK", "0"), ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0"), ("MASTER_ADDR", "127.0.0.1"),
                     ("MASTER_PORT", "29533")):
            os.environ.setdefault(k, v)  # plain `python bench.py --dist`: a one-rank group
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        # device_id binds the rank to its GPU up front (no guessed rank -> device mapping)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    P, r = dist.get_world_size(), dist.get_rank()
    local = int(os.environ.get("LOCAL_RANK", r))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    n, b, la = args.n, args.b, args.lookahead
    if torch.cuda.device_count() <= local:
        raise RuntimeError(f"rank {r}: LOCAL_RANK {local} but only {torch.cuda.device_count()} CUDA device(s) visible")
    cfg = getattr(args, "config", "c4")
    _, seed, dist_name, _, shift = (configs or {}).get(cfg, (n, 3, "uniform", b, 0.0))
    host_loc = local_columns_seeded(n, b, P, r, seed=seed, dist_name=dist_name, diag_shift=shift)  # 1/P per rank
    a0 = torch.from_numpy(host_loc).to(dev)
    a = torch.empty_like(a0)
    piv = torch.zeros(n, dtype=torch.int64, device=dev)
    kern = CudaKernels(dev)
    L = _lib.load()

    def step():
        a.copy_(a0)
        getrf_block_cyclic(a, n, b, la, kern, piv=piv)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    if clocks:
        clocks.start()
        time.sleep(0.3)
    launches0 = L.pflu_launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    lt = torch.tensor([L.pflu_launch_count() - launches0], dtype=torch.int64, device=dev)
    dist.all_reduce(lt)                      # whole job: every rank's kernel launches
    launches = int(lt.item())
    clk = clocks.stop() if clocks else None
    # every rank samples its own GPU's clocks; rank 0 reports them all
    clk_all = [None] * P
    dist.all_gather_object(clk_all, clk)
    ms_step = float(ms.item()) / args.steps
    value = lu_flops(n) / (ms_step * 1e-3) / 1e9
    peak, peak_src = fp64_peak()
    # end to end through the public API: each rank's block-cyclic columns in pinned host memory,
    # H2D, factorization, its L\U columns and the pivots back to the host (lu_factor_local)
    e2e = None
    if args.e2e_steps > 0:
        pristine = torch.from_numpy(host_loc)
        host = torch.empty(pristine.shape, dtype=torch.float64).pin_memory()
        ts = []
        for it in range(args.e2e_steps + 1):
            host.copy_(pristine)
            dist.barrier()
            t0 = time.perf_counter()
            lu, pv = lu_factor_local(host, n, b=b, lookahead=la)
            dist.barrier()
            ts.append(time.perf_counter() - t0)
        tmax = torch.tensor([sum(ts[1:]) / len(ts[1:])], dtype=torch.float64, device=dev)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        nloc = local_cols(n, b, P, r)
        e2e = {"value": lu_flops(n) / float(tmax.item()) / 1e9, "unit": unit, "h2d_bytes_per_step": n * nloc * 8,
               "d2h_bytes_per_step": n * nloc * 8 + n * 8,
               "api": "paper_1804_07017_b200.dist.lu_factor_local(pinned host block-cyclic columns) per rank"}
        del host, pristine
    if r == 0:
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": P, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload or f"C4: LUpp n={n} U[-1,1) numpy seed 3, b={b}, look-ahead {la}", "n": n, "b": b,
                       "lookahead": la, "parallelism": f"1-D block-cyclic columns over {P} GPUs, NCCL panel broadcast",
                       "l2": "inputs larger than L2; local columns restored by a D2D copy inside each step",
                       "fp64_peak_frac": value / 1e3 / (peak * P)},
            "roofline": {"bound": "tensor", "achieved": None, "peak": peak * P, "unit": "TFLOP/s",
                         "frac": value / 1e3 / (peak * P), "traffic": None, "peak_source": peak_src,
                         "note": "aggregate over ranks; per-kernel roofline is reported by the N=1 line"},
            "clocks": clk, "clocks_per_rank": clk_all, "e2e": e2e, "gpu_launches": launches, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


