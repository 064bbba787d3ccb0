"""The C ABI's multi-GPU driver (pflu_init / pflu_getrf_mg / pflu_finalize).

On the one-GPU test box the P ranks share device 0 (pflu_init(P, [0] * P)): the block-cyclic
schedule, the per-step message (panel + pivots), look-ahead across ranks and the deferred swaps all
run exactly as on P devices, with device-to-device copies instead of ncclBroadcast.  Exact mode must
be BITWISE the reference / oracle at every P; DMMA mode must give the oracle's pivots.  The NCCL
transport itself runs in a subprocess with PFLU_MG_FORCE=1 at P = 1 (a one-rank communicator).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, ROOT, bitwise_equal

pytestmark = pytest.mark.gpu

CONFIGS = json.load(open(os.path.join(GOLDEN, "configs.json")))
PIVOTS = np.load(os.path.join(GOLDEN, "configs_pivots.npz"))


@pytest.fixture
def virtual_ranks():
    from paper_1804_07017_b200 import finalize_gpus, init_gpus

    def make(P):
        init_gpus(P, [0] * P)

    yield make
    finalize_gpus()


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("lookahead", [0, 1])
def test_mg_small_golden_exact(cuda, golden_small, virtual_ranks, P, lookahead):
    from paper_1804_07017_b200 import getrf_mg

    virtual_ranks(P)
    for tag in ["grid16", "grid32", "grid80", "grid97", "u300", "la6b", "la4b7", "n257b64", "sing48", "tie4"]:
        a0 = golden_small[f"{tag}__a"]
        b, info, _ = golden_small[f"{tag}__meta"]
        if a0.shape[0] != a0.shape[1]:
            continue
        a = np.array(a0, copy=True)
        piv, inf = getrf_mg(a, int(b), lookahead, P, exact=True)
        assert inf == info, tag
        assert np.array_equal(piv, golden_small[f"{tag}__piv"]), tag
        assert bitwise_equal(a, golden_small[f"{tag}__f"]), tag


@pytest.mark.parametrize("P", [2, 4])
def test_mg_c1_exact_sha(cuda, virtual_ranks, P):
    import hashlib

    from paper_1804_07017_b200 import getrf_mg

    virtual_ranks(P)
    a = np.random.default_rng(0).uniform(-1.0, 1.0, size=(2048, 2048))
    piv, info = getrf_mg(a, 128, 1, P, exact=True)
    assert info == 0 and np.array_equal(piv, PIVOTS["c1"])
    assert hashlib.sha256(a.tobytes()).hexdigest() == CONFIGS["c1"]["sha256_factors"]


@pytest.mark.parametrize("P", [2, 3, 8])
def test_mg_dmma_pivots_and_residual(cuda, virtual_ranks, P):
    from paper_1804_07017_b200 import getrf_mg

    virtual_ranks(P)
    for n, b in [(1000, 64), (2048, 128), (777, 100)]:
        a0 = np.random.default_rng(n + P).uniform(-1, 1, (n, n))
        want, wpiv, _ = oracle.getrf(a0, b)
        for la in (0, 1):
            a = np.array(a0, copy=True)
            piv, info = getrf_mg(a, b, la, P)
            assert info == 0 and np.array_equal(piv, wpiv)
            assert oracle.lu_residual(a0, a, piv) <= 10
            assert oracle.max_rel_diff(a, want, a0) <= 1e-10


def test_mg_more_ranks_than_blocks_and_zero_columns(cuda, virtual_ranks):
    from paper_1804_07017_b200 import getrf_mg

    virtual_ranks(5)
    a0 = np.random.default_rng(7).random((64, 64))
    a0[:, [3, 17, 40]] = 0.0
    want, wpiv, winfo = oracle.getrf(a0, 16)          # 4 blocks, 5 ranks: rank 4 owns no column
    a = np.array(a0, copy=True)
    piv, info = getrf_mg(a, 16, 1, 5, exact=True)
    assert info == winfo == 4
    assert np.array_equal(piv, wpiv) and bitwise_equal(a, want)


def test_mg_trace_records(cuda, virtual_ranks):
    from paper_1804_07017_b200 import getrf_mg

    virtual_ranks(2)
    a = np.random.default_rng(1).uniform(-1, 1, (1024, 1024))
    tr = []
    getrf_mg(a, 128, 1, 2, trace=tr)
    labels = {e.label for e in tr}
    assert {"PF", "TU_R", "TU_L", "BCAST"} <= labels
    pf = [e.k for e in tr if e.label == "PF"]
    assert pf == list(range(0, 8, 2))                 # rank 0 owns the even blocks
    assert sorted(e.k for e in tr if e.label == "BCAST") == list(range(8))
    assert all(e.end >= e.start >= 0 for e in tr)


def test_lu_factor_n_gpus_in_process(cuda):
    """lu_factor(a, n_gpus=P) outside torch.distributed is the in-process C-ABI driver; with fewer
    visible GPUs than requested it fails loudly (no silent fallback to one GPU)."""
    import torch

    from paper_1804_07017_b200 import finalize_gpus, lu_factor

    a0 = np.random.default_rng(3).uniform(-1, 1, (512, 512))
    n_dev = torch.cuda.device_count()
    if n_dev >= 2:
        lu, piv = lu_factor(a0.copy(), b=64, n_gpus=2)
        assert oracle.lu_residual(a0, lu, piv) <= 10
    else:
        with pytest.raises(RuntimeError):
            lu_factor(a0.copy(), b=64, n_gpus=2)
    finalize_gpus()


def test_mg_nccl_transport_one_rank(cuda):
    """PFLU_MG_FORCE=1 routes n_gpus=1 through the multi-GPU driver with a one-rank NCCL communicator
    (ncclCommInitAll + the per-step ncclBroadcast on the panel stream): bitwise the oracle."""
    code = r"""
import numpy as np, sys
sys.path.insert(0, '.')
import oracle
from paper_1804_07017_b200 import getrf_mg, init_gpus, _lib
init_gpus(1)
assert _lib.load().pflu_mg_uses_nccl() == 1
a0 = np.random.default_rng(11).uniform(-1, 1, (700, 700))
want, wpiv, _ = oracle.getrf(a0, 64)
for la in (0, 1):
    a = a0.copy()
    piv, info = getrf_mg(a, 64, la, 1, exact=True)
    assert info == 0 and np.array_equal(piv, wpiv) and a.tobytes() == want.tobytes()
print('nccl-ok')
"""
    env = dict(os.environ, PFLU_MG_FORCE="1")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "nccl-ok" in out.stdout, out.stderr[-3000:]


def test_mg_tall_panels_multicluster_exact(cuda, virtual_ranks):
    """From 4 ranks up the owner factors panels taller than 8192 rows on the multi-cluster kernel (with the
    adaptive cluster count): n = 9472 puts the first panels there.  Exact mode must stay bitwise the oracle."""
    from paper_1804_07017_b200 import getrf_mg

    n, b, P = 9472, 256, 4
    a0 = np.random.default_rng(41).uniform(-1.0, 1.0, (n, n))
    want, wpiv, winfo = oracle.getrf(a0, b)
    virtual_ranks(P)
    a = np.array(a0, copy=True)
    piv, inf = getrf_mg(a, b, 1, P, exact=True)
    assert inf == winfo == 0
    assert np.array_equal(piv, wpiv)
    assert bitwise_equal(a, want)
