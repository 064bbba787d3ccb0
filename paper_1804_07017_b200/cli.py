"""Benchmark CLI mirroring the reference's ``python -m panelforge.bench`` for Kind.LU and Kind.QR
(pkg/src/panelforge/bench.py): sweep n, time each strategy, emit the same CSV schema.

    python -m paper_1804_07017_b200.cli --kind lu --strategy la --n-min 2048 --n-max 8192 --check

* Instances are the reference's (bench.py:85-93): ``default_rng(SeedSequence([seed, kind, n])).random``,
  uniform [0, 1), so both tools factor bitwise-identical matrices.
* Timing covers only the library call (the matrix is already on the device; generation, copies and
  checking are excluded), best of ``--reps`` after one warm-up (bench.py:120-145); CUDA events.
* ``--check`` reports ||PA - LU||_F / (n u ||A||_F) (oracle.py:78-89) computed on the GPU in row
  blocks, so it also works at C5 sizes (n = 65536) where the host residual needs ~240 GB; for QR
  ||A - QR||_F / (n u ||A||_F) (oracle.py:113-127, Q formed on the GPU by torch as the checker).
* CSV: ``kind,strategy,n,b,threads,seconds,gflops,residual`` (bench.py:32, 219-234); the
  ``threads`` column carries the GPU count.
* Strategies: mtb (look-ahead 0), la (look-ahead 1, dynamic tile schedule: the block scheduler hands
  the panel's SMs back to pending GEMM tiles), la-static (look-ahead 1, SM-partitioned: the panel's
  SMs stay with the panel chain -- the reference's non-malleable LA), la-mb (partitioned + a join grid
  that puts the panel's SMs on the trailing GEMM's remaining tiles after PF(k+1): the reference's
  malleable team, runtime.py:99-113).  rtm is not offered (out of scope; racy in the reference,
  SURVEY.md App. A.4).
"""
from __future__ import annotations

import argparse
import sys
from dataclasses import dataclass

import numpy as np

CSV_HEADER = "kind,strategy,n,b,threads,seconds,gflops,residual"
_KINDS = ("lu", "qr", "gemm")
# strategy -> (CSV label, look-ahead depth, pflu_options.malleable)
_STRATEGIES = {"mtb": ("MTB", 0, 0), "la": ("LA", 1, 0), "la-static": ("LA_STATIC", 1, 1), "la-mb": ("LA_MB", 1, 2)}
UNIT_ROUNDOFF = 2.0 ** -53


@dataclass(frozen=True)
class BenchRecord:
    kind: str
    strategy: str
    n: int
    b: int
    threads: int
    seconds: float
    gflops: float
    residual: float | None = None


def make_instance(seed: int, kind: str, n: int) -> np.ndarray:
    """The reference's problem matrix for (seed, kind, n) (bench.py:85-93), row-major."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, _KINDS.index(kind), n]))
    return rng.random((n, n))


def lu_residual_gpu(a0, lu, piv, block: int = 4096) -> float:
    """||P A - L U||_F / (n u ||A||_F) on the GPU (torch fp64 matmul used as the checker)."""
    import torch

    dev = lu.device
    n = a0.shape[1]
    m = a0.shape[0]
    pv = piv.cpu().numpy() if hasattr(piv, "cpu") else np.asarray(piv)
    pm = np.arange(m)
    for i, r in enumerate(pv):
        if r != i:
            pm[i], pm[r] = pm[r], pm[i]
    perm = torch.from_numpy(pm).to(dev)
    upper = torch.triu(lu[:n])
    err2 = 0.0
    for r0 in range(0, m, block):
        r1 = min(m, r0 + block)
        low = torch.tril(lu[r0:r1, :n], diagonal=r0 - 1)
        idx = torch.arange(r0, min(r1, n), device=dev)
        low[idx - r0, idx] = 1.0
        d = a0.index_select(0, perm[r0:r1]) - low @ upper
        err2 += float((d * d).sum())
    norm_a = float(torch.linalg.norm(a0))
    err = err2 ** 0.5
    return err if norm_a == 0.0 else err / (max(n, 1) * UNIT_ROUNDOFF * norm_a)


def time_factor(a_host: np.ndarray, b: int, lookahead: int, reps: int, check: bool, malleable: int = 0):
    import torch

    from .api import getrf_device

    dev = torch.device("cuda", torch.cuda.current_device())
    pristine = torch.from_numpy(np.ascontiguousarray(a_host)).to(dev)
    work = torch.empty_like(pristine)
    piv = torch.empty(pristine.shape[1], dtype=torch.int64, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def once():
        work.copy_(pristine)
        torch.cuda.synchronize()
        e0.record()
        getrf_device(work, b, lookahead, piv=piv, malleable=malleable)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3

    once()  # warm-up (bench.py:137)
    best = min(once() for _ in range(max(1, reps)))
    residual = lu_residual_gpu(pristine, work, piv) if check else None
    return best, residual


def qr_residual_gpu(a0, f, tau) -> float:
    """||A - Q R||_F / (n u ||A||_F) on the GPU, Q = H_1 ... H_n formed by torch (checker only)."""
    import torch

    m, n = a0.shape
    v = torch.tril(f, -1) + torch.eye(m, n, device=f.device, dtype=f.dtype)
    q = torch.linalg.householder_product(v, tau)
    norm_a = float(torch.linalg.norm(a0))
    err = float(torch.linalg.norm(a0 - q @ torch.triu(f[:n])))
    return err if norm_a == 0.0 else err / (max(n, 1) * UNIT_ROUNDOFF * norm_a)


def time_factor_qr(a_host: np.ndarray, b: int, lookahead: int, reps: int, check: bool):
    import torch

    from .api import geqrf_device

    dev = torch.device("cuda", torch.cuda.current_device())
    pristine = torch.from_numpy(np.ascontiguousarray(a_host)).to(dev)
    work = torch.empty_like(pristine)
    tau = torch.zeros(pristine.shape[1], dtype=torch.float64, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def once():
        work.copy_(pristine)
        torch.cuda.synchronize()
        e0.record()
        geqrf_device(work, b, lookahead, tau=tau)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3

    once()
    best = min(once() for _ in range(max(1, reps)))
    residual = qr_residual_gpu(pristine, work, tau) if check else None
    return best, residual


def run_sweep(kind: str, strategies, sizes, b: int, reps: int, seed: int, check: bool):
    import torch

    from .api import Kind, flops

    if kind not in ("lu", "qr"):
        raise ValueError(f"--kind {kind}: only lu and qr are implemented on the B200 (GEMM studies are out of scope)")
    gpus = 1 if torch.cuda.is_available() else 0
    records = []
    for n in sizes:
        a = make_instance(seed, kind, n)
        for s in strategies:
            label, la, mall = _STRATEGIES[s]
            if kind == "qr":
                seconds, residual = time_factor_qr(a, b, la, reps, check)
                fl = flops(Kind.QR, n)
            else:
                seconds, residual = time_factor(a, b, la, reps, check, malleable=mall)
                fl = flops(Kind.LU, n)
            records.append(BenchRecord(kind.upper(), label, n, b, gpus, seconds, fl / seconds / 1e9, residual))
    return records


def emit_csv(records, sink) -> None:
    own = isinstance(sink, str)
    f = open(sink, "w", encoding="ascii") if own else sink
    try:
        f.write(CSV_HEADER + "\n")
        for r in records:
            res = "" if r.residual is None else repr(r.residual)
            f.write(f"{r.kind},{r.strategy},{r.n},{r.b},{r.threads},{r.seconds!r},{r.gflops!r},{res}\n")
    finally:
        if own:
            f.close()


def parse_csv(text: str):
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0] != CSV_HEADER:
        raise ValueError("missing or unexpected CSV header")
    out = []
    for ln in lines[1:]:
        kind, strategy, n, b, threads, seconds, gflops, residual = ln.split(",")
        out.append(BenchRecord(kind, strategy, int(n), int(b), int(threads), float(seconds), float(gflops),
                               None if residual == "" else float(residual)))
    return out


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_1804_07017_b200.cli",
                                description="Sweep matrix sizes and report LU GFLOPS per strategy as CSV (B200).")
    p.add_argument("--kind", choices=_KINDS, default="lu")
    p.add_argument("--strategy", choices=list(_STRATEGIES) + ["all"], default="all")
    p.add_argument("--n-min", type=int, default=256)
    p.add_argument("--n-max", type=int, default=4096)
    p.add_argument("--n-step", type=int, default=256)
    p.add_argument("--b", type=int, default=192, help="panel/block size")
    p.add_argument("--threads", type=int, default=None, help="accepted for compatibility (ignored: GPU)")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--check", action="store_true", help="backward error on the GPU (not timed)")
    p.add_argument("--csv", default="stdout", help="output path, or 'stdout'")
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    if args.n_min < 1 or args.n_max < args.n_min or args.n_step < 1:
        raise SystemExit("invalid size range")
    sizes = list(range(args.n_min, args.n_max + 1, args.n_step))
    strategies = list(_STRATEGIES) if args.strategy == "all" else [args.strategy]
    records = run_sweep(args.kind, strategies, sizes, args.b, args.reps, args.seed, args.check)
    emit_csv(records, sys.stdout if args.csv == "stdout" else args.csv)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
