"""Multi-process tests of the 1-D block-cyclic driver (paper_1804_07017_b200.dist), gloo on CPU.

The product schedule runs unchanged; kernels come from the CPU oracle (tests/dist_oracle_backend.py),
so the distributed factorization must be BITWISE equal to the single-process reference result
(the per-element operation order does not depend on the column distribution).
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, b, lookahead, seed, out_dir, singular):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dist_oracle_backend import OracleKernels
    from paper_1804_07017_b200 import dist as pd

    a = np.random.default_rng(seed).uniform(-1.0, 1.0, (n, n))
    if singular:
        a[:, 5] = 0.0
    loc = pd.scatter_columns(torch.from_numpy(a), b, world, rank)
    piv, info = pd.getrf_block_cyclic(loc, n, b, lookahead, OracleKernels())
    lu = pd.allgather_columns(loc, n, b)
    if rank == 0:
        np.save(os.path.join(out_dir, "lu.npy"), lu.numpy())
        np.save(os.path.join(out_dir, "piv.npy"), piv.numpy())
        np.save(os.path.join(out_dir, "info.npy"), np.array([info]))
    dist.barrier()
    dist.destroy_process_group()


def _run(tmp_path, world, n, b, lookahead, seed=0, singular=False):
    mp.spawn(_worker, args=(world, _free_port(), n, b, lookahead, seed, str(tmp_path), singular), nprocs=world,
             join=True)
    return (np.load(tmp_path / "lu.npy"), np.load(tmp_path / "piv.npy"), int(np.load(tmp_path / "info.npy")[0]))


@pytest.mark.parametrize("world,n,b,lookahead", [(2, 96, 16, 1), (2, 100, 16, 0), (3, 101, 8, 1), (2, 64, 64, 1),
                                                 (3, 40, 16, 1), (4, 150, 16, 1), (4, 72, 8, 0)])
def test_block_cyclic_matches_reference_bitwise(tmp_path, world, n, b, lookahead):
    import oracle

    a = np.random.default_rng(0).uniform(-1.0, 1.0, (n, n))
    ref, rpiv, rinfo = oracle.getrf(a, b)
    lu, piv, info = _run(tmp_path, world, n, b, lookahead)
    assert info == rinfo == 0
    assert np.array_equal(piv, rpiv)
    assert lu.tobytes() == ref.tobytes()


def _trace_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dist_oracle_backend import OracleKernels
    from paper_1804_07017_b200 import dist as pd

    n, b = 96, 16
    a = np.random.default_rng(0).uniform(-1.0, 1.0, (n, n))
    for la in (0, 1):
        loc = pd.scatter_columns(torch.from_numpy(a), b, world, rank)
        tr = []
        pd.getrf_block_cyclic(loc, n, b, la, OracleKernels(), trace=tr)
        np.save(os.path.join(out_dir, f"trace_{la}_{rank}.npy"),
                np.array([(e.label, e.k, e.start, e.end) for e in tr], dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_block_cyclic_trace_records(tmp_path):
    """The distributed driver's trace hook: every rank records BCAST for every step, PF for the
    blocks it owns, TU_R (look-ahead 1) / TU (look-ahead 0) per step, TU_L where it owns block k+1."""
    world = 2
    mp.spawn(_trace_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for la in (0, 1):
        for rank in range(world):
            recs = np.load(tmp_path / f"trace_{la}_{rank}.npy", allow_pickle=True)
            by = {}
            for label, k, s_, e_ in recs:
                by.setdefault(label, []).append(int(k))
                assert e_ >= s_
            assert sorted(by["BCAST"]) == list(range(6))
            assert sorted(by["PF"]) == list(range(rank, 6, world))
            if la == 0:
                assert sorted(by["TU"]) == list(range(6))
            else:
                assert sorted(by["TU_R"]) == list(range(6))
                assert sorted(by["TU_L"]) == [k for k in range(5) if (k + 1) % world == rank]


def test_block_cyclic_singular_info(tmp_path):
    import oracle

    a = np.random.default_rng(0).uniform(-1.0, 1.0, (48, 48))
    a[:, 5] = 0.0
    ref, rpiv, rinfo = oracle.getrf(a, 16)
    lu, piv, info = _run(tmp_path, 2, 48, 16, 1, singular=True)
    assert info == rinfo == 6
    assert np.array_equal(piv, rpiv)
    assert lu.tobytes() == ref.tobytes()


def test_block_cyclic_bookkeeping():
    from paper_1804_07017_b200 import dist as pd

    n, b = 1000, 64
    for P in (1, 2, 3, 8):
        assert sum(pd.local_cols(n, b, P, r) for r in range(P)) == n
        a = torch.arange(n * n, dtype=torch.float64).view(n, n)
        parts = [pd.scatter_columns(a, b, P, r) for r in range(P)]
        assert torch.equal(pd.gather_columns(parts, n, b), a)
        for r in range(P):
            for k in range(pd.num_blocks(n, b)):
                if k % P == r:
                    lc = pd.local_col_of_block(k, b, P)
                    assert torch.equal(parts[r][:, lc: lc + min(b, n - k * b)], a[:, k * b: min(n, (k + 1) * b)])
                    assert pd.local_cols_before(k, n, b, P, r) == lc


@pytest.mark.parametrize("dist_name,seed", [("uniform", 3), ("normal", 2)])
def test_local_columns_seeded_match_full_matrix(dist_name, seed):
    """Chunked per-rank generation == the block-cyclic columns of the full seeded BASELINE matrix."""
    sys.path.insert(0, ROOT)
    from paper_1804_07017_b200 import dist as pd

    n, b = 530, 64
    g = np.random.default_rng(seed)
    full = g.uniform(-1.0, 1.0, (n, n)) if dist_name == "uniform" else g.standard_normal((n, n))
    for P in (1, 3):
        for r in range(P):
            loc = pd.local_columns_seeded(n, b, P, r, seed, dist_name, chunk_rows=100)
            assert loc.tobytes() == pd.scatter_columns(torch.from_numpy(full), b, P, r).numpy().tobytes()


def _qr_worker(rank, world, port, n, b, lookahead, seed, out_dir, zero_col=-1):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dist_oracle_backend import OracleKernels
    from paper_1804_07017_b200 import dist as pd

    a = np.random.default_rng(seed).uniform(-1.0, 1.0, (n, n))
    if zero_col >= 0:
        a[:, zero_col] = 0.0   # a zero column stays zero under every reflector: tau = 0 there
    loc = pd.scatter_columns(torch.from_numpy(a), b, world, rank)
    tau = pd.geqrf_block_cyclic(loc, n, b, lookahead, OracleKernels())
    f = pd.allgather_columns(loc, n, b)
    if rank == 0:
        np.save(os.path.join(out_dir, "f.npy"), f.numpy())
        np.save(os.path.join(out_dir, "tau.npy"), tau.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,b,lookahead,zero_col", [(2, 96, 16, 1, -1), (2, 100, 16, 0, -1), (3, 101, 8, 1, -1),
                                                          (4, 150, 16, 1, -1), (2, 64, 16, 1, 0), (3, 80, 8, 0, 21)])
def test_qr_block_cyclic_matches_oracle_bitwise(tmp_path, world, n, b, lookahead, zero_col):
    """The distributed Householder QR (same schedule, oracle kernels) is bitwise the single-process
    oracle: every column's operation sequence is independent of the column distribution (also with a
    null reflector, tau = 0, in a column owned by a non-zero rank)."""
    import oracle

    mp.spawn(_qr_worker, args=(world, _free_port(), n, b, lookahead, 7, str(tmp_path), zero_col), nprocs=world,
             join=True)
    f, tau = np.load(tmp_path / "f.npy"), np.load(tmp_path / "tau.npy")
    a = np.random.default_rng(7).uniform(-1.0, 1.0, (n, n))
    if zero_col >= 0:
        a[:, zero_col] = 0.0
        assert tau[zero_col] == 0.0
    rf, rtau = oracle.geqrf(a, b)
    assert f.tobytes() == rf.tobytes() and tau.tobytes() == rtau.tobytes()


def _emu_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dist_oracle_backend import OracleKernels
    from paper_1804_07017_b200 import dist as pd

    n, b = 96, 16
    a = torch.from_numpy(np.random.default_rng(0).uniform(-1.0, 1.0, (n, n)))
    tr = []
    pd.getrf_block_cyclic(a.clone(), n, b, 1, OracleKernels(), trace=tr, emulate=4)
    np.save(os.path.join(out_dir, "emu.npy"), np.array([(e.label, e.k) for e in tr], dtype=object), allow_pickle=True)
    dist.destroy_process_group()


def test_block_cyclic_emulation_mode(tmp_path):
    """emulate=Q (the scaling model on dist.py's own k-loop): one rank factors every panel (PF and TU_L on
    every step, as each step's owner) and runs TU_R on its share; refused at world size > 1."""
    mp.spawn(_emu_worker, args=(1, _free_port(), str(tmp_path)), nprocs=1, join=True)
    recs = np.load(tmp_path / "emu.npy", allow_pickle=True)
    labels = [str(r[0]) for r in recs]
    assert labels.count("PF") == 6 and labels.count("TU_L") == 5 and labels.count("TU_R") == 6
