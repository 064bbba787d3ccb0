"""The block-cyclic driver with the product CUDA backend (GPU box, one GPU).

World size 1 runs in-process (NCCL); world size 2 runs two processes on cuda:0 with gloo carrying
the panel broadcasts (the ranks' kernels never wait on each other -- only the host collective
synchronises them).  Exact mode must be bitwise equal to the oracle, DMMA mode must match pivots
and backward error.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, backend, n, b, lookahead, exact, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    from paper_1804_07017_b200 import dist as pd

    dev = torch.device("cuda:0")
    a = np.random.default_rng(4).uniform(-1.0, 1.0, (n, n))
    loc = pd.scatter_columns(torch.from_numpy(a), b, world, rank).to(dev)
    piv, info = pd.getrf_block_cyclic(loc, n, b, lookahead, pd.CudaKernels(dev, exact=exact))
    lu = pd.allgather_columns(loc, n, b)
    if rank == 0:
        np.save(os.path.join(out_dir, "lu.npy"), lu.cpu().numpy())
        np.save(os.path.join(out_dir, "piv.npy"), piv.cpu().numpy())
        np.save(os.path.join(out_dir, "info.npy"), np.array([info]))
    dist.barrier()
    dist.destroy_process_group()


def _run(tmp_path, world, backend, n, b, lookahead, exact):
    mp.spawn(_worker, args=(world, _free_port(), backend, n, b, lookahead, exact, str(tmp_path)), nprocs=world,
             join=True)
    return np.load(tmp_path / "lu.npy"), np.load(tmp_path / "piv.npy"), int(np.load(tmp_path / "info.npy")[0])


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo")])
@pytest.mark.parametrize("n,b,lookahead", [(700, 64, 1), (513, 128, 0), (2048, 256, 1)])
def test_dist_cuda_exact_bitwise(cuda, tmp_path, world, backend, n, b, lookahead):
    a = np.random.default_rng(4).uniform(-1.0, 1.0, (n, n))
    ref, rpiv, _ = oracle.getrf(a, b)
    lu, piv, info = _run(tmp_path, world, backend, n, b, lookahead, True)
    assert info == 0
    assert np.array_equal(piv, rpiv)
    assert lu.tobytes() == ref.tobytes()


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo")])
def test_dist_cuda_dmma(cuda, tmp_path, world, backend):
    n, b = 1500, 128
    a = np.random.default_rng(4).uniform(-1.0, 1.0, (n, n))
    ref, rpiv, _ = oracle.getrf(a, b)
    lu, piv, info = _run(tmp_path, world, backend, n, b, 1, False)
    assert np.array_equal(piv, rpiv)
    assert oracle.lu_residual(a, lu, piv) <= 10
    assert oracle.max_rel_diff(lu, ref, a) <= 1e-8


def _worker_api(rank, world, port, backend, n, b, gather, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["LOCAL_RANK"] = "0"
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    from paper_1804_07017_b200 import dist as pd

    a = np.random.default_rng(8).uniform(-1.0, 1.0, (n, n))
    host = torch.from_numpy(a.copy()).pin_memory()
    lu, piv, info = pd.lu_factor_dist(host, b=b, lookahead=1, exact=True, return_info=True, gather=gather)
    out = lu.numpy() if isinstance(lu, torch.Tensor) else np.asarray(lu)
    np.save(os.path.join(out_dir, f"lu{rank}.npy"), out)
    np.save(os.path.join(out_dir, f"piv{rank}.npy"), piv.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("gather", ["all", "local"])
def test_lu_factor_dist_api(cuda, tmp_path, gather):
    from paper_1804_07017_b200 import dist as pd

    n, b, world = 700, 64, 2
    a = np.random.default_rng(8).uniform(-1.0, 1.0, (n, n))
    ref, rpiv, _ = oracle.getrf(a, b)
    mp.spawn(_worker_api, args=(world, _free_port(), "gloo", n, b, gather, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        lu = np.load(tmp_path / f"lu{r}.npy")
        assert np.array_equal(np.load(tmp_path / f"piv{r}.npy"), rpiv)
        if gather == "all":
            assert lu.tobytes() == ref.tobytes()
        else:   # the rank's own block-cyclic columns hold the factors
            for j in pd.local_blocks(n, b, world, r):
                sl = slice(j * b, min(n, (j + 1) * b))
                assert lu[:, sl].tobytes() == np.ascontiguousarray(ref[:, sl]).tobytes()


def _worker_local(rank, world, port, n, b, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["LOCAL_RANK"] = "0"
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1804_07017_b200 import dist as pd

    loc = torch.from_numpy(pd.local_columns_seeded(n, b, world, rank, seed=9)).pin_memory()
    out, piv, info = pd.lu_factor_local(loc, n, b=b, lookahead=1, exact=True, return_info=True)
    np.save(os.path.join(out_dir, f"loc{rank}.npy"), out.numpy())
    np.save(os.path.join(out_dir, f"piv{rank}.npy"), np.asarray(piv))
    dist.barrier()
    dist.destroy_process_group()


def test_lu_factor_local_api(cuda, tmp_path):
    """ScaLAPACK-style distributed input: each rank passes only its block-cyclic columns."""
    from paper_1804_07017_b200 import dist as pd

    n, b, world = 600, 64, 2
    a = np.random.default_rng(9).uniform(-1.0, 1.0, (n, n))
    ref, rpiv, _ = oracle.getrf(a, b)
    mp.spawn(_worker_local, args=(world, _free_port(), n, b, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"piv{r}.npy"), rpiv)
        want = pd.scatter_columns(torch.from_numpy(ref), b, world, r).numpy()
        assert np.load(tmp_path / f"loc{r}.npy").tobytes() == want.tobytes()


def _qr_worker(rank, world, port, backend, n, b, lookahead, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    from paper_1804_07017_b200 import dist as pd

    dev = torch.device("cuda:0")
    a = np.random.default_rng(5).uniform(-1.0, 1.0, (n, n))
    loc = pd.scatter_columns(torch.from_numpy(a), b, world, rank).to(dev)
    tau = pd.geqrf_block_cyclic(loc, n, b, lookahead, pd.CudaKernels(dev))
    f = pd.allgather_columns(loc, n, b)
    if rank == 0:
        np.save(os.path.join(out_dir, "f.npy"), f.cpu().numpy())
        np.save(os.path.join(out_dir, "tau.npy"), tau.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo")])
@pytest.mark.parametrize("n,b,lookahead", [(700, 64, 1), (513, 128, 0), (2048, 256, 1)])
def test_dist_cuda_qr(cuda, tmp_path, world, backend, n, b, lookahead):
    """Block-cyclic Householder QR with the CUDA kernels: factors and tau within 1e-10 of the oracle,
    backward error / orthogonality <= 10."""
    mp.spawn(_qr_worker, args=(world, _free_port(), backend, n, b, lookahead, str(tmp_path)), nprocs=world,
             join=True)
    f, tau = np.load(tmp_path / "f.npy"), np.load(tmp_path / "tau.npy")
    a = np.random.default_rng(5).uniform(-1.0, 1.0, (n, n))
    rf, rtau = oracle.geqrf(a, b)
    assert np.abs(f - rf).max() / np.abs(a).max() <= 1e-10
    assert np.abs(tau - rtau).max() <= 1e-10
    back, orth = oracle.qr_residual(a, f, tau)
    assert back <= 10 and orth <= 10


def _trace_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1804_07017_b200 import dist as pd

    dev = torch.device("cuda:0")
    n, b = 1024, 128
    a = np.random.default_rng(4).uniform(-1.0, 1.0, (n, n))
    loc = pd.scatter_columns(torch.from_numpy(a), b, world, rank).to(dev)
    tr = []
    pd.getrf_block_cyclic(loc, n, b, 1, pd.CudaKernels(dev), trace=tr)
    np.save(os.path.join(out_dir, f"tr_{rank}.npy"), np.array([(e.label, e.k, e.start, e.end) for e in tr],
                                                              dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_dist_cuda_trace(cuda, tmp_path):
    """CUDA-event trace of the distributed driver (2 ranks on cuda:0, gloo): PF on the owned blocks,
    BCAST / TU_R on every step, TU_L where the rank owns block k+1; times non-negative, ordered."""
    mp.spawn(_trace_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for rank in range(2):
        recs = np.load(tmp_path / f"tr_{rank}.npy", allow_pickle=True)
        by = {}
        for label, k, s_, e_ in recs:
            by.setdefault(label, []).append(int(k))
            assert 0 <= s_ <= e_
        assert sorted(by["PF"]) == list(range(rank, 8, 2))
        assert sorted(by["BCAST"]) == list(range(8)) and sorted(by["TU_R"]) == list(range(8))


@pytest.mark.parametrize("ranks", [1, 8])
def test_dist_tall_panel_kernel_choice_bitwise(cuda, ranks):
    """CudaKernels.panel sends panels taller than grid_rows to the multi-cluster kernel -- two clusters while
    the rank's share of the trailing update would outlast the panel (ranks = 1 here), all of them otherwise
    (ranks = 8): both must be bitwise the oracle's lu_unb on the panel (exact mode)."""
    import torch

    import oracle
    from paper_1804_07017_b200 import _lib
    from paper_1804_07017_b200 import dist as pd

    m, w = 20000, 256
    p0 = np.random.default_rng(97).uniform(-1.0, 1.0, (m, w))
    want, wpiv, winfo = oracle.lu_unb(p0.copy())
    kern = pd.CudaKernels(cuda, exact=True, grid_rows=8192)
    kern.ranks = ranks
    assert kern.opt_grid.panel_kernel == _lib.PANEL_MCLUSTER and kern.opt_grid2.panel_ctas == 32
    x = torch.from_numpy(p0).to(cuda)
    piv = torch.zeros(w, dtype=torch.int64, device=cuda)
    with kern.stream("P"):
        kern.panel(x, m, 0, 0, w, piv)
    torch.cuda.synchronize()
    assert winfo == 0
    assert np.array_equal(piv.cpu().numpy(), wpiv)
    assert x.cpu().numpy().tobytes() == want.tobytes()
