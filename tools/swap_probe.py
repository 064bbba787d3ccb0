"""Standalone timing of the pivot plan + fused laswp/trsm at the C4 step-0 shape (and ncu target)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ncols = int(sys.argv[3]) if len(sys.argv) > 3 else n - nb
L = _lib.load()
dev = torch.device("cuda:0")
a = torch.rand(n, nb + ncols, dtype=torch.float64, device=dev)
rng = np.random.default_rng(0)
piv = torch.from_numpy(np.array([rng.integers(k, n) for k in range(nb)], dtype=np.int64)).to(dev)
st = torch.cuda.current_stream().cuda_stream
ld = nb + ncols
f = lambda: _lib.check(L.pflu_swap_trsm(a.data_ptr(), ld, 0, 0, nb, piv.data_ptr(), nb, nb + ncols, st), "st")  # noqa
g = lambda: _lib.check(L.pflu_laswp(a.data_ptr(), ld, nb, nb + ncols, piv.data_ptr(), 0, nb, st), "sw")  # noqa
for name, fn in (("swap+trsm", f), ("laswp only", g)):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} n={n} nb={nb} ncols={ncols}: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
