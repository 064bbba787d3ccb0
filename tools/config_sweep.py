"""Throughput of every BASELINE.json config on one B200 (device-resident, CUDA events, best of reps).
Writes the JSON list to argv[1] (default profiles/r02_configs.json)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import getrf_device  # noqa: E402

dev = torch.device("cuda:0")


def mat(name):
    if name == "C1":
        return np.random.default_rng(0).uniform(-1, 1, (2048, 2048))
    if name in ("C2", "C2s"):
        a = np.random.default_rng(1).uniform(-1, 1, (8192, 8192))
        if name == "C2s":
            a[np.diag_indices(8192)] += 8192.0
        return a
    if name == "C3":
        return np.random.default_rng(2).standard_normal((16384, 16384))
    if name == "C4":
        return np.random.default_rng(3).uniform(-1, 1, (32768, 32768))
    if name == "C5":
        return np.random.default_rng(4).standard_normal((65536, 65536))


def timeit(a0, b, la, reps):
    a = torch.empty_like(a0)
    ts = []
    for r in range(reps + 1):
        a.copy_(a0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        getrf_device(a, b, la)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    return min(ts)


out = []
plan = [("C1", [128], [1, 0], 10), ("C2", [256], [1, 0], 5), ("C2s", [256], [1], 5),
        ("C3", [64, 128, 256, 512], [0, 1], 3), ("C4", [256], [1, 0], 2), ("C5", [512], [1], 1)]
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None  # e.g. C1,C2,C3
for name, bs, las, reps in plan:
    if only and name not in only:
        continue
    a0 = torch.from_numpy(mat(name)).to(dev)
    n = a0.shape[0]
    for b in bs:
        for la in las:
            ms = timeit(a0, b, la, reps)
            rec = {"config": name, "n": n, "b": b, "lookahead": la, "ms": round(ms, 3),
                   "tflops": round(2 * n ** 3 / 3 / ms / 1e9, 2), "frac_of_37.17": round(2 * n ** 3 / 3 / ms / 1e9 / 37.17, 3)}
            print(json.dumps(rec), flush=True)
            out.append(rec)
    del a0
    torch.cuda.empty_cache()
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_configs.json", "w"), indent=1)
