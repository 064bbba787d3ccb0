"""Panel-chain gap analysis of one factorization (run with PFLU_EMU_RANKS=8 for the 8-rank model): where the
time on the chain PF(k) -> TU_L(k) -> PF(k+1) goes besides the PF and TU_L kernels themselves."""
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
pf = {ev.k: ev for ev in tr if ev.label == "PF"}
tl = {ev.k: ev for ev in tr if ev.label == "TU_L"}
steps = max(pf) + 1
t0 = min(ev.start for ev in tr)
t1 = max(ev.end for ev in tr)
g1 = sum((tl[k].start - pf[k].end) * 1e3 for k in range(steps) if k in tl)
g2 = sum((pf[k + 1].start - tl[k].end) * 1e3 for k in range(steps) if k in tl and k + 1 in pf)
print(f"n={n} b={b}: total {tot:.1f} ms; trace span {(t1 - t0) * 1e3:.1f}; sum PF {sum((e.end - e.start) for e in pf.values()) * 1e3:.1f}, "
      f"sum TU_L {sum((e.end - e.start) for e in tl.values()) * 1e3:.1f}; gaps PF->TU_L {g1:.1f}, TU_L->PF {g2:.1f}; "
      f"head (start->PF0 start) {(pf[0].start - t0) * 1e3:.2f}, tail (last PF end -> end) {(t1 - pf[steps - 1].end) * 1e3:.2f}")
for k in list(range(3)) + list(range(steps // 2, steps // 2 + 3)) + list(range(steps - 4, steps - 1)):
    if k in tl and k + 1 in pf:
        print(f"  k={k:3d} PF {1e3 * (pf[k].end - pf[k].start):.3f}  gap {1e3 * (tl[k].start - pf[k].end):.3f}  TU_L {1e3 * (tl[k].end - tl[k].start):.3f}"
              f"  gap {1e3 * (pf[k + 1].start - tl[k].end):.3f}")
