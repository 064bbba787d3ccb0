"""QR throughput on one B200 (device-resident, CUDA events): 4/3 n^3 / t for n x n inputs.
Usage: python tools/qr_bench.py [n ...]  (env QR_B, QR_LA to pick block size / look-ahead)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_07017_b200 import qr_factor  # noqa: E402


def run(n, b, la, reps=2):
    if n > 32768:  # generated on the device (the host generator takes minutes at this size)
        g = torch.Generator(device="cuda").manual_seed(4)
        a0 = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    else:
        a0 = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, (n, n))).cuda()
    w = a0.clone()
    qr_factor(w, b=b, lookahead=la)  # warm-up (workspaces)
    best = 1e30
    for _ in range(reps):
        w.copy_(a0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        qr_factor(w, b=b, lookahead=la)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    fl = 4.0 * n ** 3 / 3.0
    return {"n": n, "b": b, "lookahead": la, "ms": round(best, 2), "tflops": round(fl / best / 1e9, 3)}


if __name__ == "__main__":
    ns = [int(x) for x in sys.argv[1:]] or [4096, 8192, 16384]
    for n in ns:
        for la in [int(x) for x in os.environ.get("QR_LA", "0,1").split(",")]:
            print(json.dumps(run(n, int(os.environ.get("QR_B", "256")), la)), flush=True)
