"""LA (SM-partitioned) vs LA_MB (partitioned + join grid) vs the dynamic tile schedule, device-resident
factorizations timed with CUDA events (best of reps).  Usage: python tools/malleable_probe.py [n ...]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import getrf_device  # noqa: E402

sizes = [int(x) for x in sys.argv[1:]] or [8192, 16384, 32768]
dev = torch.device("cuda:0")
for n in sizes:
    b = 256
    d0 = torch.empty(n, n, dtype=torch.float64, device=dev).uniform_(-1, 1)
    x = torch.empty_like(d0)
    row = {"n": n, "b": b}
    import os

    modes = [(0, "dynamic"), (1, "la_static"), (2, "la_mb")]
    if os.environ.get("PROBE_DYNAMIC_ONLY"):
        modes = modes[:1]
    for mode, name in modes:
        best = 1e9
        for rep in range(3):
            x.copy_(d0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            getrf_device(x, b, 1, malleable=mode)
            e1.record()
            torch.cuda.synchronize()
            if rep > 0:
                best = min(best, e0.elapsed_time(e1))
        row[name + "_ms"] = round(best, 2)
        row[name + "_tflops"] = round(2 * n ** 3 / 3 / (best * 1e-3) / 1e12, 2)
    print(json.dumps(row), flush=True)
