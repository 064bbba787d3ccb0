"""One panel factorization (after warm-up) for ncu launch lists."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import _lib  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
w = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ctas = int(sys.argv[3]) if len(sys.argv) > 3 else 0
leaf = int(sys.argv[4]) if len(sys.argv) > 4 else 0
kern = int(sys.argv[5]) if len(sys.argv) > 5 else 0
L = _lib.load()
dev = torch.device("cuda:0")
x0 = torch.rand(m, w, dtype=torch.float64, device=dev) * 2 - 1
x = x0.clone()
piv = torch.zeros(w, dtype=torch.int64, device=dev)
info = ctypes.c_int64(0)
opt = _lib.options(exact=False, panel_ctas=ctas, leaf_width=leaf, panel_kernel=kern)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    x.copy_(x0)
    _lib.check(L.pflu_panel(x.data_ptr(), w, m, 0, 0, w, piv.data_ptr(), ctypes.byref(info), st, ctypes.byref(opt)), "p")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
x.copy_(x0)
e0.record()
_lib.check(L.pflu_panel(x.data_ptr(), w, m, 0, 0, w, piv.data_ptr(), ctypes.byref(info), st, ctypes.byref(opt)), "p")
e1.record()
torch.cuda.synchronize()
print(f"panel m={m} w={w} ctas={ctas} leaf={leaf}: {e0.elapsed_time(e1):.3f} ms", flush=True)
