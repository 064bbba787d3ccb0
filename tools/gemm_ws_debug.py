"""Locate wrong tiles of a GEMM variant (debug): C = C - A B on shape M x N x K in the factorization's
layout; prints bad 128x64 tiles and bad k-stage hypotheses."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import _lib  # noqa: E402

L = _lib.load()
dev = torch.device("cuda:0")
M, N, K, pad = (int(x) for x in sys.argv[1:5])
for rep in range(3):
    g = torch.Generator(device=dev).manual_seed(M + N + K)
    buf = torch.randn(M + K, K + N + pad, dtype=torch.float64, device=dev, generator=g)
    c = buf[K:K + M, K:K + N]
    a = buf[K:K + M, 0:K].clone()
    b = buf[0:K, K:K + N].clone()
    want = c - a @ b
    _lib.check(L.pflu_gemm_update(c.data_ptr(), c.stride(0), buf[K:, 0:K].data_ptr(), buf.stride(0),
                                  buf[0:K, K:].data_ptr(), buf.stride(0), M, N, K, 0,
                                  torch.cuda.current_stream().cuda_stream), "gemm")
    torch.cuda.synchronize()
    err = (c - want).abs() > 1e-9
    bad = err.nonzero()
    print(f"rep {rep}: bad elements {len(bad)} of {M * N}", flush=True)
    if len(bad):
        tiles = torch.unique(torch.stack([bad[:, 0] // 128, bad[:, 1] // 64], 1), dim=0)
        print("  bad tiles", len(tiles), tiles[:12].tolist())
        r0, c0 = (int(x) for x in bad[0])
        # which k range explains the error: compare with partial products
        d = (c - want)[r0, c0].item()
        for ks in range(0, K, 16):
            part = (a[r0, ks:ks + 16] @ b[ks:ks + 16, c0]).item()
            if abs(abs(part) - abs(d)) < 1e-9 * max(1, abs(d)):
                print("  error at", r0, c0, "matches k-block", ks, "sign", d / part)
        rows = torch.unique(bad[:, 0] % 128)
        cols = torch.unique(bad[:, 1] % 64)
        print("  rows in tile", rows[:40].tolist(), "cols in tile", cols[:70].tolist())
