"""Scaling model for the 1-D block-cyclic multi-GPU LU on ONE GPU (gpurun gives one).

For P ranks, the per-step critical path of dist.py is TU_L(k) + PF(k+1) on the owner of block k+1,
then the panel broadcast; every rank meanwhile runs TU_R(k) on ~1/P of the trailing columns.  With
PFLU_EMU_RANKS=P, libpflu's depth-1 schedule runs exactly that on one GPU: this rank factors EVERY
panel (as its owner would, on the dist.py panel kernel choice) but updates only 1/P of each trailing
matrix.  T_P(model) = emulated time + sum over steps of the panel broadcast ((n - kb) * b * 8 bytes at
the NVLink bandwidth given, plus a fixed latency).  This is a MODEL, not a multi-GPU measurement.

    python tools/emu_scaling.py --n 32768 --b 256 --ranks 1,2,4,8 [--pf-kernel 3]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child_dist(n, b, reps, P):
    """The same model on dist.py's own k-loop (getrf_block_cyclic(..., emulate=P)) -- the code a
    torchrun job runs -- in a one-rank process group on this GPU."""
    import socket

    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    from paper_1804_07017_b200 import dist as pd

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("gloo", rank=0, world_size=1)
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    a0 = torch.rand((n, n), dtype=torch.float64, device=dev, generator=g) * 2 - 1
    a = torch.empty_like(a0)
    piv = torch.empty(n, dtype=torch.int64, device=dev)
    kern = pd.CudaKernels(dev)
    best = None
    for it in range(reps + 1):
        a.copy_(a0)
        tr = []
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pd.getrf_block_cyclic(a, n, b, 1, kern, piv=piv, trace=tr, emulate=P)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if it == 0:
            continue
        rec = {"ms": ms, "pf_ms": sum((e.end - e.start) * 1e3 for e in tr if e.label == "PF"),
               "tul_ms": sum((e.end - e.start) * 1e3 for e in tr if e.label == "TU_L"),
               "gemm_ms": sum((e.end - e.start) * 1e3 for e in tr if e.label == "TU_R")}
        if best is None or ms < best["ms"]:
            best = rec
    print("EMU " + json.dumps(best), flush=True)
    dist.destroy_process_group()


def child(n, b, reps):
    import torch

    sys.path.insert(0, ROOT)
    from paper_1804_07017_b200 import getrf_device

    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    a0 = torch.rand((n, n), dtype=torch.float64, device=dev, generator=g) * 2 - 1
    a = torch.empty_like(a0)
    piv = torch.empty(n, dtype=torch.int64, device=dev)
    best = None
    for it in range(reps + 1):
        a.copy_(a0)
        tr = []
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        getrf_device(a, b, 1, piv=piv, trace=tr)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if it == 0:
            continue
        pf = sum((e.end - e.start) * 1e3 for e in tr if e.label == "PF")
        tul = sum((e.end - e.start) * 1e3 for e in tr if e.label == "TU_L")
        gem = sum((e.end - e.start) * 1e3 for e in tr if e.label == "GEMM")
        rec = {"ms": ms, "pf_ms": pf, "tul_ms": tul, "gemm_ms": gem}
        if best is None or ms < best["ms"]:
            best = rec
    print("EMU " + json.dumps(best), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--b", type=int, default=256)
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--pf-kernel", type=int, default=-1, help="force PFLU_PF_KERNEL (3 = recursive panel)")
    ap.add_argument("--nvlink-gbs", type=float, default=700.0, help="effective broadcast bandwidth per GPU")
    ap.add_argument("--bcast-lat-us", type=float, default=25.0, help="fixed cost per step (2 broadcasts + pack)")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--driver", default="cpp", choices=["cpp", "dist"],
                    help="cpp: libpflu's single-GPU schedule with PFLU_EMU_RANKS; dist: dist.py's own k-loop "
                         "(getrf_block_cyclic(emulate=P)), the code torchrun runs")
    ap.add_argument("--emu-p", type=int, default=1, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.child:
        if args.driver == "dist":
            child_dist(args.n, args.b, args.reps, args.emu_p)
        else:
            child(args.n, args.b, args.reps)
        return
    n, b = args.n, args.b
    bcast_ms = sum(((n - k * b) * b * 8 / (args.nvlink_gbs * 1e9) + args.bcast_lat_us * 1e-6) * 1e3
                   for k in range(1, -(-n // b)))
    flops = 2.0 * n ** 3 / 3.0
    t1 = None
    for P in [int(x) for x in args.ranks.split(",")]:
        env = dict(os.environ)
        if args.driver == "cpp":
            env["PFLU_EMU_RANKS"] = str(P)
        if args.pf_kernel >= 0:
            env["PFLU_PF_KERNEL"] = str(args.pf_kernel)
        out = subprocess.run([sys.executable, __file__, "--child", "--n", str(n), "--b", str(b), "--reps", str(args.reps),
                              "--driver", args.driver, "--emu-p", str(P)],
                             env=env, capture_output=True, text=True, cwd=ROOT)
        line = [ln for ln in out.stdout.splitlines() if ln.startswith("EMU ")]
        if not line:
            print(out.stdout[-2000:], out.stderr[-2000:])
            continue
        r = json.loads(line[-1][4:])
        t = r["ms"] + (bcast_ms if P > 1 else 0.0)
        if P == 1:
            t1 = t
        eff = t1 / (P * t) if t1 else None
        print(json.dumps({"driver": args.driver, "P": P, "n": n, "b": b, "pf_kernel": args.pf_kernel, "emulated_ms": r["ms"],
                          "bcast_model_ms": bcast_ms if P > 1 else 0.0, "model_ms": t,
                          "model_tflops": flops / (t * 1e-3) / 1e12, "model_efficiency": eff,
                          "sum_pf_ms": r["pf_ms"], "sum_tul_ms": r["tul_ms"], "sum_gemm_ms": r["gemm_ms"]}), flush=True)


if __name__ == "__main__":
    main()
