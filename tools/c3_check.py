import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1804_07017_b200 import lu_factor
P = np.load("tests/golden/configs_pivots.npz")["c3"]
a0 = np.random.default_rng(2).standard_normal((16384, 16384))
for b in (int(x) for x in sys.argv[1:] or [512]):
    for exact in (False, True):
        lu, piv = lu_factor(a0.copy(), b=b, lookahead=1, exact=exact)
        bad = np.nonzero(piv != P)[0]
        print(b, "exact" if exact else "dmma", "mismatches", len(bad), "first", bad[:5].tolist(), flush=True)
