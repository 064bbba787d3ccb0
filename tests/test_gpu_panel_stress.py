"""Stress of the panel kernel's zero-pivot path, exact mode, BITWISE
against the oracle's lu_unb (reference _jit.py:154-187; an exactly-zero pivot column is left as is
and the next column's search runs from the tile, _jit.py:171-174).

Zero columns at many positions -- first / middle / last column of a leaf, consecutive zero columns,
a zero first column, every column zero -- on the grid (LL exchange) and cluster (DSMEM) kernels
with 1..16 CTAs and leaf widths 8 / 16 / 32, each case repeated PFLU_STRESS_REPEATS times (default
2; tools/panel_hazard.sh runs 50 against the exact-as-template build).
"""
import ctypes
import os

import numpy as np
import pytest

import oracle
from conftest import bitwise_equal

pytestmark = pytest.mark.gpu

REPEATS = int(os.environ.get("PFLU_STRESS_REPEATS", "2"))

ZERO_PATTERNS = {
    "none": [],
    "first": [0],
    "j5": [5],
    "leaf_edges": [7, 8, 15, 16],
    "consecutive": [3, 4, 5],
    "pairs": [1, 2, 9, 10, 30, 31],
    "last": [-1],
    "every_other": "odd",
    "all": "all",
}


def _zero_cols(w, pat):
    if pat == "odd":
        return list(range(1, w, 2))
    if pat == "all":
        return list(range(w))
    return sorted({(c if c >= 0 else w + c) for c in pat if (c if c >= 0 else w + c) < w})


CASES = [(48, 16), (48, 48), (200, 32), (1000, 64), (3000, 32)]


@pytest.mark.parametrize("m,w", CASES)
@pytest.mark.parametrize("pat", sorted(ZERO_PATTERNS))
@pytest.mark.parametrize("kernel", [1, 2], ids=["grid", "cluster"])
def test_panel_zero_pivots_bitwise(cuda, m, w, pat, kernel):
    import torch
    from paper_1804_07017_b200 import _lib as lb

    rng = np.random.default_rng(m * 131 + w)
    p0 = rng.random((m, w))
    zc = _zero_cols(w, ZERO_PATTERNS[pat])
    p0[:, zc] = 0.0
    want, wpiv, winfo = oracle.lu_unb(p0.copy())
    L = lb.load()
    st = torch.cuda.current_stream().cuda_stream
    for ctas in (1, 2, 3, 7, 16):
        if ctas > m:
            continue
        for leaf in (8, 16, 32):
            for rep in range(REPEATS):
                x = torch.from_numpy(p0).to(cuda)
                piv = torch.full((w,), -7, dtype=torch.int64, device=cuda)
                info = ctypes.c_int64(0)
                opt = lb.options(exact=True, panel_ctas=ctas, leaf_width=leaf, panel_kernel=kernel)
                rc = L.pflu_panel(x.data_ptr(), w, m, 0, 0, w, piv.data_ptr(), ctypes.byref(info), st,
                                  ctypes.byref(opt))
                if kernel == 2 and rc == 3:
                    continue  # does not fit one cluster at this CTA count
                lb.check(rc, "pflu_panel")
                torch.cuda.synchronize()
                got_piv = piv.cpu().numpy()[: len(wpiv)]
                tag = f"ctas={ctas} leaf={leaf} rep={rep} zero_cols={zc[:8]}"
                assert np.array_equal(got_piv, wpiv), f"pivots differ ({tag}): first at " \
                    f"{int(np.nonzero(got_piv != wpiv)[0][0])}"
                assert info.value == winfo, tag
                assert bitwise_equal(x.cpu().numpy(), want), tag


@pytest.mark.parametrize("lookahead", [0, 1])
def test_getrf_zero_columns_exact(cuda, lookahead):
    """Full factorizations with zero columns inside and across panel boundaries: bitwise = oracle,
    info = first zero column (1-based)."""
    from paper_1804_07017_b200 import lu_factor

    for n, b, zc in [(48, 16, [5]), (300, 64, [0, 63, 64, 65]), (777, 128, [100, 101, 102, 500]),
                     (1024, 256, list(range(256, 288)))]:
        a0 = np.random.default_rng(n).random((n, n))
        a0[:, zc] = 0.0
        want, wpiv, winfo = oracle.getrf(a0, b)
        for rep in range(REPEATS):
            lu, piv, info = lu_factor(a0.copy(), b=b, lookahead=lookahead, exact=True, return_info=True)
            assert info == winfo == zc[0] + 1
            assert np.array_equal(piv, wpiv)
            assert bitwise_equal(lu, want)
