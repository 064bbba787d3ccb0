"""Trailing-update GEMM variants (PFLU_GEMM_WS / PFLU_GEMM_VARIANT, read when libpflu loads): parity
against a torch fp64 matmul on ragged shapes, then TFLOP/s at C4-like shapes inside an n x n matrix
(A = L21 and B = U12 are views with lda = n, exactly as in the factorization).
Usage: python tools/gemm_ws_probe.py [n] [reps]   (one process per variant: run under env)"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
L = _lib.load()
dev = torch.device("cuda:0")
st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
tag = f"ws={os.environ.get('PFLU_GEMM_WS', '-')} var={os.environ.get('PFLU_GEMM_VARIANT', '-')}"


def upd(c, a, b):
    M, N = c.shape
    K = a.shape[1]
    _lib.check(L.pflu_gemm_update(c.data_ptr(), c.stride(0), a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0),
                                  M, N, K, 0, st()), "gemm")


worst = 0.0
for (M, N, K, ld) in [(1, 1, 1, 2), (129, 65, 16, 130), (3001, 2999, 256, 3002), (1000, 700, 100, 1000),
                      (4096, 4096, 256, 4352), (257, 4000, 256, 4000), (5000, 64, 256, 5000)]:
    g = torch.Generator(device=dev).manual_seed(M + N + K)
    buf = torch.randn(M + K, K + N + (ld % 16), dtype=torch.float64, device=dev, generator=g)
    c = buf[K:K + M, K:K + N]   # the factorization's layout: L21 left of C, U12 above it
    a = buf[K:K + M, 0:K]
    b = buf[0:K, K:K + N]
    want = c - a @ b
    a_, b_ = a.clone(), b.clone()
    bound = 2 * K * 2.0 ** -53 * (a_.abs() @ b_.abs()) + 1e-300
    upd(c, a, b)
    torch.cuda.synchronize()
    r = float(((c - want).abs() / bound).max())
    worst = max(worst, r)
    print(f"{tag} parity {M}x{N}x{K} ld={ld}: max |err| / (2 K u |a||b|) = {r:.3f}", flush=True)
assert worst <= 1.0, worst
big = torch.empty(n, n, dtype=torch.float64, device=dev)
big.uniform_(-1, 1)
for k0, kk in [(256, 256), (n // 2, 256), (3 * n // 4, 256)]:
    c = big[k0:, k0:]
    a = big[k0:, k0 - kk:k0]
    b = big[k0 - kk:k0, k0:]
    for _ in range(2):
        upd(c, a, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        upd(c, a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    M, N = c.shape
    print(f"{tag} gemm {M}x{N}x{kk} (lda={n}): {ms:.3f} ms  {2 * M * N * kk / ms / 1e9:.1f} TFLOP/s", flush=True)
