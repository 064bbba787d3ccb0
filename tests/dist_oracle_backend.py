"""CPU kernel backend for the block-cyclic driver, built on the oracle (TEST INFRASTRUCTURE).

Runs paper_1804_07017_b200.dist.getrf_block_cyclic -- the product schedule -- on torch CPU
tensors under gloo, with every kernel call served by oracle/pflu_oracle.c through raw pointers and
leading dimensions.  Streams and events are no-ops (program order is a valid serialisation of the
schedule).  Used only by tests/test_dist.py.
"""
import contextlib
import ctypes

import numpy as np
import torch

import oracle

_d = ctypes.POINTER(ctypes.c_double)
_i = ctypes.POINTER(ctypes.c_int64)


def _dp(t, off=0):
    return ctypes.cast(t.data_ptr() + 8 * off, _d)


def _ip(t, off=0):
    return ctypes.cast(t.data_ptr() + 8 * off, _i)


class OracleKernels:
    is_cuda = False

    def __init__(self):
        self.L = oracle.lib()
        self.info = 0

    def stream(self, which):
        return contextlib.nullcontext()

    def event(self):
        return None

    def record(self, ev, which):
        pass

    def wait(self, ev, which):
        pass

    def begin(self):
        pass

    def join(self):
        pass

    def info_reset(self):
        self.info = 0

    def info_read(self):
        return self.info

    def panel(self, a, m, d, col, w, piv):
        ld = a.stride(0)
        k = min(w, m - d)
        tmp = torch.zeros(k, dtype=torch.int64)
        info = self.L.orc_lu_unb(_dp(a, d * ld + col), m - d, w, ld, _ip(tmp), -1)
        piv[d: d + k] = tmp + d
        if info and (self.info == 0 or d + info < self.info):
            self.info = d + info

    def plan(self, piv, d, nb, plan):
        plan[0] = d
        plan[1: 1 + nb] = piv[d: d + nb]

    def swap_trsm(self, a, d, nb, plan, c0, c1, l11=None):
        if c1 <= c0:
            return
        ld = a.stride(0)
        full = torch.zeros(d + nb, dtype=torch.int64)
        full[d:] = plan[1: 1 + nb]
        self.L.orc_laswp(_dp(a), ld, c0, c1, _ip(full), d, d + nb)
        if l11 is not None:
            self.L.orc_trsm_llnu(_dp(l11), l11.stride(0), nb, _dp(a, d * ld + c0), ld, c1 - c0)

    def gemm(self, c, a, b):
        m, n = c.shape
        k = a.shape[1]
        if m and n and k:
            self.L.orc_gemm_sub(_dp(c), c.stride(0), _dp(a), a.stride(0), _dp(b), b.stride(0), m, n, k)

    # Householder QR: the oracle's qr_unb / larft / block reflector on the same views
    def qr_panel(self, a, m, d, col, w, tau):
        ld = a.stride(0)
        tmp = torch.zeros(w, dtype=torch.float64)
        self.L.orc_qr_unb(_dp(a, d * ld + col), m - d, w, ld, _dp(tmp))
        tau.copy_(tmp)

    def qr_apply(self, v, tau, c):
        mp, k = v.shape
        nc = c.shape[1]
        if nc == 0 or mp == 0:
            return
        vv = v.contiguous()
        tt = tau.contiguous()
        t = torch.zeros((k, k), dtype=torch.float64)
        self.L.orc_larft(_dp(vv), mp, k, vv.stride(0), _dp(tt), _dp(t))
        self.L.orc_apply_block_reflector(_dp(vv), mp, k, vv.stride(0), _dp(t), _dp(c), nc, c.stride(0))
