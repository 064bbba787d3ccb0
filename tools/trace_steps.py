"""Per-step breakdown of one factorization from the library's CUDA-event trace."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import getrf_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
b = int(sys.argv[2]) if len(sys.argv) > 2 else 256
la = int(sys.argv[3]) if len(sys.argv) > 3 else 1
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
    getrf_device(a, b, la, trace=tr)
    e1.record()
    torch.cuda.synchronize()
tot = e0.elapsed_time(e1)
by = {}
for ev in tr:  # chunked TU_R: several records per (label, k) -> span from first start to last end
    if (ev.label, ev.k) in by:
        o = by[(ev.label, ev.k)]
        by[(ev.label, ev.k)] = type(ev)(ev.label, ev.k, ev.j, min(o.start, ev.start), max(o.end, ev.end), None, o.flop + ev.flop)
    else:
        by[(ev.label, ev.k)] = ev
steps = max(ev.k for ev in tr) + 1
lab_r = "TU_R" if la else "TU"
gemm_ms = sum((by[k].end - by[k].start) * 1e3 for k in by if k[0] == "GEMM")
pf_ms = sum((ev.end - ev.start) * 1e3 for ev in tr if ev.label == "PF")
tul_ms = sum((ev.end - ev.start) * 1e3 for ev in tr if ev.label == "TU_L")
tur_ms = sum((by[k].end - by[k].start) * 1e3 for k in by if k[0] == lab_r)
gaps = 0.0
rows = []
for k in range(steps):
    r = by.get((lab_r, k))
    rn = by.get((lab_r, k + 1))
    pf = by.get(("PF", k + 1))
    tl = by.get(("TU_L", k))
    gm = by.get(("GEMM", k))
    gap = (rn.start - r.end) * 1e3 if (r and rn) else 0.0
    gaps += max(0.0, gap)
    rows.append((k, (r.end - r.start) * 1e3 if r else 0, (gm.end - gm.start) * 1e3 if gm else 0,
                 (tl.end - tl.start) * 1e3 if tl else 0, (pf.end - pf.start) * 1e3 if pf else 0, gap))
print(f"n={n} b={b} la={la}: total {tot:.1f} ms = {2 * n**3 / 3 / tot / 1e9:.1f} TFLOP/s; sum TU_R {tur_ms:.1f}, GEMM {gemm_ms:.1f}, "
      f"TU_L {tul_ms:.1f}, PF {pf_ms:.1f}, gaps between TU_R {gaps:.1f} ms")
print(" k    TU_R    GEMM    TU_L     PF(k+1)  gap")
for row in rows[:4] + rows[steps // 2: steps // 2 + 2] + rows[-24:]:
    print(" %3d %7.3f %7.3f %7.3f %7.3f %7.3f" % row)
