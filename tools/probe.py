"""Quick perf probe of the individual kernels and the full factorization (GPU box)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import _lib, lu_factor, getrf_device  # noqa: E402

L = _lib.load()
dev = torch.device("cuda:0")
st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), float(np.median(ts))


def gemm(M, N, K, exact):
    c = torch.randn(M, N, dtype=torch.float64, device=dev)
    a = torch.randn(M, K, dtype=torch.float64, device=dev)
    b = torch.randn(K, N, dtype=torch.float64, device=dev)
    f = lambda: _lib.check(L.pflu_gemm_update(c.data_ptr(), N, a.data_ptr(), K, b.data_ptr(), N, M, N, K, exact, st()), "g")  # noqa
    tmin, tmed = timeit(f)
    print(f"gemm M={M} N={N} K={K} exact={exact}: {tmin:.3f} ms  {2*M*N*K/tmin/1e9:.1f} GFLOP/s (med {2*M*N*K/tmed/1e9:.1f})", flush=True)


def panel(m, w, ctas=0, leaf=0):
    x0 = torch.rand(m, w, dtype=torch.float64, device=dev) * 2 - 1
    x = x0.clone()
    piv = torch.zeros(w, dtype=torch.int64, device=dev)
    info = ctypes.c_int64(0)
    opt = _lib.options(exact=False, panel_ctas=ctas, leaf_width=leaf)

    def f():
        x.copy_(x0)
        _lib.check(L.pflu_panel(x.data_ptr(), w, m, 0, 0, w, piv.data_ptr(), ctypes.byref(info), st(), ctypes.byref(opt)), "p")
    tmin, tmed = timeit(f, reps=3, warm=1)
    print(f"panel m={m} w={w} ctas={ctas} leaf={leaf}: {tmin:.3f} ms (incl. copy)", flush=True)


def getrf(n, b, la, exact=False, seed=3):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    a0 = torch.rand(n, n, dtype=torch.float64, device=dev, generator=g) * 2 - 1
    a = torch.empty_like(a0)
    piv = torch.empty(n, dtype=torch.int64, device=dev)
    ts = []
    for r in range(3):
        a.copy_(a0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        getrf_device(a, b, la, exact=exact, piv=piv)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts)
    fl = 2 * n ** 3 / 3
    print(f"getrf n={n} b={b} la={la} exact={exact}: {t:.1f} ms  {fl/t/1e9:.1f} GFLOP/s  ({fl/t/1e9/37100:.3f} of 37.1 TF)  all={['%.1f'%x for x in ts]}", flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "gemm"):
        gemm(8192, 8192, 256, 0)
        gemm(32512, 32512, 256, 0)
        gemm(16384, 16384, 512, 0)
        gemm(8192, 8192, 256, 1)
    if what in ("all", "panel"):
        for m in (2048, 8192, 32768):
            panel(m, 256)
        panel(32768, 256, 32)
    if what in ("all", "getrf"):
        getrf(2048, 128, 1)
        getrf(8192, 256, 0)
        getrf(8192, 256, 1)
        getrf(16384, 256, 1)
        getrf(32768, 256, 0)
        getrf(32768, 256, 1)
