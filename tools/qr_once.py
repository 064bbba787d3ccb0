"""One QR factorization (device-resident) for ncu launch lists: python tools/qr_once.py n b lookahead."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07017_b200 import qr_factor  # noqa: E402

n, b, la = (int(x) for x in (sys.argv[1:] + ["8192", "256", "1"][len(sys.argv) - 1:]))
a = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, (n, n))).cuda()
qr_factor(a, b=b, lookahead=la)
torch.cuda.synchronize()
print("ok", n, b, la)
