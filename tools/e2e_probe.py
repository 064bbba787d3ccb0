import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_1804_07017_b200 import lu_factor
n = 32768
rng = np.random.default_rng(3)
pinned = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
host = pinned.numpy()
a0 = rng.uniform(-1, 1, (n, n))
for it in range(3):
    np.copyto(host, a0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lu, pv = lu_factor(host, b=256, lookahead=1)
    print(f"wall {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
