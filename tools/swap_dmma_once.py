"""One fast-mode swap+TRSM (pivot plan, inverted 32x32 diagonal blocks, DMMA solve) at the C4 step-0
shape and one deferred left-swap launch (pure row permutation) at a mid-factorization shape -- the ncu
targets for the TRSM FP64-pipe and laswp HBM evidence (tools/prof_round.sh)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 256
left = int(sys.argv[3]) if len(sys.argv) > 3 else n // 2      # columns of the left swaps
L = _lib.load()
dev = torch.device("cuda:0")
a = torch.rand(n, n, dtype=torch.float64, device=dev)
rng = np.random.default_rng(0)
st = torch.cuda.current_stream().cuda_stream


def setup(d):
    piv = torch.zeros(n, dtype=torch.int64, device=dev)
    piv[d: d + nb] = torch.from_numpy(np.array([rng.integers(d + k, n) for k in range(nb)], dtype=np.int64))
    plan = torch.empty(1 + 3 * nb, dtype=torch.int64, device=dev)
    _lib.check(L.pflu_pivot_plan(piv.data_ptr(), d, nb, plan.data_ptr(), st), "plan")
    return plan


plan0 = setup(0)                      # step 0: swap + solve of columns [nb, n) (the C4 step-0 width)
inv = torch.empty(((nb + 31) // 32) * 1024, dtype=torch.float64, device=dev)
_lib.check(L.pflu_diag_inv(a.data_ptr(), n, nb, inv.data_ptr(), st), "inv")
dl = left                             # a mid step: its deferred left swaps on columns [0, left)
plan1 = setup(dl)


def trsm():
    _lib.check(L.pflu_swap_trsm_inv(a.data_ptr(), n, 0, nb, plan0.data_ptr(), nb, n, a.data_ptr(), n,
                                    inv.data_ptr(), st), "trsm")


def lswap():
    _lib.check(L.pflu_swap_trsm_plan(a.data_ptr(), n, dl, nb, plan1.data_ptr(), 0, left, None, n, st), "lswap")


for name, fn in (("swap+trsm (DMMA)", trsm), ("left swaps", lswap)):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
