"""Component timing of the QR path on one B200 (CUDA events, device buffers):
panel (pflu_qr_panel), larft (pflu_larft, includes its host-side transpose), block reflector apply."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07017_b200 import _lib  # noqa: E402

L = _lib.load()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for mp in [int(x) for x in (sys.argv[1:] or ["4096", "16384", "32768"])]:
    k = 256
    a0 = torch.rand(mp, k, dtype=torch.float64, device="cuda") * 2 - 1
    a = a0.clone()
    tau = torch.zeros(k, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def panel():
        a.copy_(a0)
        assert L.pflu_qr_panel(a.data_ptr(), k, mp, 0, 0, k, tau.data_ptr(), st) == 0

    t_copy = timed(lambda: a.copy_(a0))
    t_panel = timed(panel) - t_copy
    t32 = torch.zeros(mp, 32, dtype=torch.float64, device="cuda")
    t32.copy_(a0[:, :32])
    a32 = t32.clone()

    def leaf():
        a32.copy_(t32)
        assert L.pflu_qr_panel(a32.data_ptr(), 32, mp, 0, 0, 32, tau.data_ptr(), st) == 0

    t_leaf = timed(leaf) - timed(lambda: a32.copy_(t32))
    panel()
    T = torch.zeros(k, k, dtype=torch.float64, device="cuda")
    t_larft = timed(lambda: L.pflu_larft(a.data_ptr(), k, mp, k, tau.data_ptr(), T.data_ptr(), k, st))
    nc = mp - k
    c = torch.rand(mp, nc, dtype=torch.float64, device="cuda")
    t_apply = timed(lambda: L.pflu_apply_block_reflector(a.data_ptr(), k, mp, k, tau.data_ptr(), c.data_ptr(), nc, nc, st))
    print(json.dumps({"mp": mp, "panel_ms": round(t_panel, 3), "leaf32_ms": round(t_leaf, 3),
                      "larft_ms(incl host T transpose)": round(t_larft, 3),
                      "build+apply_ms": round(t_apply, 3), "apply_tflops": round(4.0 * mp * nc * k / t_apply / 1e9, 2)}),
          flush=True)
