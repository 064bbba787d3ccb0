"""How much of the look-ahead run's swap + U12-solve time is NOT hidden under a trailing GEMM: the union of
the TU_R spans (swap + solve + GEMM per chunk) minus the union of the GEMM spans, from the library's trace."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import getrf_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
b = int(sys.argv[2]) if len(sys.argv) > 2 else 256
dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(3)
a0 = torch.rand(n, n, dtype=torch.float64, device=dev, generator=g) * 2 - 1
a = torch.empty_like(a0)
for it in range(2):
    a.copy_(a0)
    tr = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    getrf_device(a, b, 1, trace=tr)
    e1.record()
    torch.cuda.synchronize()
tot = e0.elapsed_time(e1)


def union(iv):
    iv = sorted(iv)
    out = []
    for s, e in iv:
        if out and s <= out[-1][1]:
            out[-1][1] = max(out[-1][1], e)
        else:
            out.append([s, e])
    return out


def length(u):
    return sum(e - s for s, e in u) * 1e3


labels = sorted({ev.label for ev in tr})
ug = union([(ev.start, ev.end) for ev in tr if ev.label == "GEMM"])
ur = union([(ev.start, ev.end) for ev in tr if ev.label in ("TU_R", "GEMM")])
ul = union([(ev.start, ev.end) for ev in tr if ev.label in ("TU_R", "GEMM", "TU_L")])
print(f"n={n} b={b}: total {tot:.1f} ms; labels {labels}; GEMM-busy {length(ug):.1f} ms; TU_R-busy {length(ur):.1f} ms; "
      f"exposed swap+solve (TU_R minus GEMM) {length(ur) - length(ug):.2f} ms; with TU_L {length(ul) - length(ug):.2f} ms")
