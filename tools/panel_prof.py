"""Per-phase clock breakdown of the persistent panel kernel (CTA 0), via pflu_debug_panel_profile."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import _lib  # noqa: E402

NAMES = ["load", "warp_best#2", "finish+publish", "top(after G)", "gather(w0)", "barrier G", "wb+swaps", "sync", "U-trsm", "blk-update", "pass1 loop", "warp_best#1", "red barrier", "g:wait keys", "g:reduce", "g:pull"]
m = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
w = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ctas = int(sys.argv[3]) if len(sys.argv) > 3 else 0
leaf = int(sys.argv[4]) if len(sys.argv) > 4 else 0
exact = int(sys.argv[5]) if len(sys.argv) > 5 else 0
kern = int(sys.argv[6]) if len(sys.argv) > 6 else 0
import os
if os.environ.get("PFLU_LIB_PATH"):
    _lib.LIB_PATH = os.environ["PFLU_LIB_PATH"]
L = _lib.load()
L.pflu_debug_panel_profile.argtypes = [ctypes.c_void_p]
dev = torch.device("cuda:0")
prof = torch.zeros(8192 + 256 * 64 * 4, dtype=torch.int64, device=dev)
x0 = torch.rand(m, w, dtype=torch.float64, device=dev) * 2 - 1
x = x0.clone()
piv = torch.zeros(w, dtype=torch.int64, device=dev)
info = ctypes.c_int64(0)
opt = _lib.options(exact=bool(exact), panel_ctas=ctas, leaf_width=leaf, panel_kernel=kern)
st = torch.cuda.current_stream().cuda_stream
run = lambda: _lib.check(L.pflu_panel(x.data_ptr(), w, m, 0, 0, w, piv.data_ptr(), ctypes.byref(info), st, ctypes.byref(opt)), "p")  # noqa
for _ in range(2):
    x.copy_(x0)
    run()
torch.cuda.synchronize()
x.copy_(x0)
L.pflu_debug_panel_profile(prof.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
L.pflu_debug_panel_profile(None)
ms = e0.elapsed_time(e1)
PP = prof.cpu()[:4096].view(256, 16)
P = PP[:, :16]
nz = int((P.sum(1) > 0).sum())
P = P[:nz].double() / 1965.0
print(f"panel m={m} w={w} ctas={ctas} W={leaf} exact={exact}: {ms:.3f} ms; {nz} CTAs; phases us (min/mean/max over CTAs):")
for i, n in enumerate(NAMES):
    col = P[:, i]
    print(f"   {n:12s} {col.min():8.0f} {col.mean():8.0f} {col.max():8.0f}   argmax CTA {int(col.argmax())}")


G = prof.cpu()[4096:4096 + w].double() / 1965.0
WP = prof.cpu()[4096 + 256:4096 + 256 + 4096].view(256, 16)[:nz].double() / 1965.0
if float(WP.sum()) > 0:
    print("   v2 worker (warp 1 lane 0): 5 = pass 2 + rest, 3 = barrier wait + top, 10 = pass 1, 11 = warp arg-max, 2 = finish + publish")
    for i in (5, 3, 10, 11, 2):
        col = WP[:, i]
        print(f"   worker[{i:2d}]   {col.min():8.0f} {col.mean():8.0f} {col.max():8.0f}")
    print("   v2 exchange warp rows above: gather(w0) = post + loop, g:wait keys, g:reduce, g:pull")

print(f"   gather us: mean {G.mean():.2f} median {G.median():.2f} max {G.max():.1f}")


