"""Diagnose a panel-kernel mismatch vs the oracle: print differing entries (hex) and pivots.
Usage: PFLU_LIB_PATH=... python tools/panel_hazard_diag.py m w pattern ctas leaf kernel"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
from paper_1804_07017_b200 import _lib as lb  # noqa: E402

m, w, pat, ctas, leaf, kernel = sys.argv[1:7]
m, w, ctas, leaf, kernel = int(m), int(w), int(ctas), int(leaf), int(kernel)
p0 = np.random.default_rng(m * 131 + w).random((m, w))
if pat == "all":
    p0[:] = 0.0
elif pat == "sing48":
    p0 = np.load("tests/golden/small_cases.npz")["sing48__a"][:, :w].copy()
    m = p0.shape[0]
elif pat != "none":
    p0[:, [int(c) for c in pat.split(",")]] = 0.0
want, wpiv, winfo = oracle.lu_unb(p0.copy())
x = torch.from_numpy(np.ascontiguousarray(p0)).cuda()
piv = torch.full((w,), -7, dtype=torch.int64, device="cuda")
info = ctypes.c_int64(0)
opt = lb.options(exact=True, panel_ctas=ctas, leaf_width=leaf, panel_kernel=kernel)
lb.check(lb.load().pflu_panel(x.data_ptr(), w, m, 0, 0, w, piv.data_ptr(), ctypes.byref(info),
                              torch.cuda.current_stream().cuda_stream, ctypes.byref(opt)), "panel")
torch.cuda.synchronize()
got = x.cpu().numpy()
gp = piv.cpu().numpy()[: len(wpiv)]
print("info", info.value, winfo, "piv equal", np.array_equal(gp, wpiv))
if not np.array_equal(gp, wpiv):
    d = np.nonzero(gp != wpiv)[0]
    print("piv mismatch cols", d[:10], "got", gp[d[:10]], "want", wpiv[d[:10]])
diff = np.nonzero(got.view(np.int64) != want.view(np.int64))
print("n diff", len(diff[0]))
for i, j in list(zip(*diff))[:8]:
    print(i, j, got[i, j], want[i, j], got[i, j].tobytes().hex(), want[i, j].tobytes().hex())
