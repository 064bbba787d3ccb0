"""A few launches of the trailing-update GEMM (C -= A*B) for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import _lib  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
K = int(sys.argv[3]) if len(sys.argv) > 3 else 256
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
L = _lib.load()
dev = torch.device("cuda:0")
c = torch.randn(M, N, dtype=torch.float64, device=dev)
a = torch.randn(M, K, dtype=torch.float64, device=dev)
b = torch.randn(K, N, dtype=torch.float64, device=dev)
st = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(reps + 2):
    if i == 2:
        e0.record()
    _lib.check(L.pflu_gemm_update(c.data_ptr(), N, a.data_ptr(), K, b.data_ptr(), N, M, N, K, 0, st), "g")
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"gemm {M}x{N}x{K}: {ms:.3f} ms  {2 * M * N * K / ms / 1e9:.1f} TFLOP/s", flush=True)
if len(sys.argv) > 5 and sys.argv[5] == "cublas":
    for i in range(reps + 2):
        if i == 2:
            e0.record()
        torch.addmm(c, a, b, alpha=-1.0, out=c)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cublas addmm {M}x{N}x{K}: {ms:.3f} ms  {2 * M * N * K / ms / 1e9:.1f} TFLOP/s", flush=True)
