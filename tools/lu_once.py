"""One device-resident factorization after a warm-up (for ncu launch lists).  Usage: lu_once.py n b"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import getrf_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
b = int(sys.argv[2]) if len(sys.argv) > 2 else 256
d0 = torch.empty(n, n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
x = d0.clone()
getrf_device(x, b, 1)
x.copy_(d0)
torch.cuda.synchronize()
getrf_device(x, b, 1)
torch.cuda.synchronize()
print("ok")
