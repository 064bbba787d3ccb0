#!/usr/bin/env python
"""Benchmark: LU with partial pivoting (BASELINE.json metric: FP64 GFLOP/s = (2/3 n^3)/t).

Workload (BASELINE.json configs[3], "C4"): n = 32768 float64, entries U[-1,1) from
numpy default_rng(3), b = 256, look-ahead depth 1.  One "step" = one full factorization of that
matrix on the GPU, inputs already resident in HBM (the factorization is in place, so the pristine
matrix is copied back with a device-to-device copy for every step -- inside the timed region: into
the idle one of two work buffers on a side stream while the other is factored, or, when three
copies do not fit (C5), at the start of every step; 8.6 GB > L2, so no L2 flush is needed).  Timed
with CUDA events on the launching stream.

--gpus N > 1 (under torchrun, one rank per GPU): 1-D block-cyclic column distribution with an
NCCL panel + pivot broadcast (paper_1804_07017_b200.dist); value = whole-job GFLOP/s.

--impl reference: the reference algorithm's CPU implementation -- the oracle port
(oracle/pflu_oracle.c, bit-for-bit the reference's arithmetic) with every host thread -- timed
on a bounded sample of the same workload: the first blocked step of C4 (panel + laswp + trsm +
trailing GEMM of the n=32768 matrix).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LU-pp FP64 GFLOP/s (2/3*n^3/t)"
UNIT = "GFLOP/s"


def lu_flops(n: int) -> float:
    return 2.0 * n ** 3 / 3.0


def fp64_peak() -> tuple[float, str]:
    """FP64 roofline denominator: the measured DMMA peak (profiles/r01_fp64_peak.jsonl, measured
    on this pool's B200 with tools/fp64_peak.cu; MEASURED_PEAKS.json carries no FP64 figure)."""
    path = os.path.join(ROOT, "profiles", "r01_fp64_peak.jsonl")
    best = 0.0
    try:
        for line in open(path):
            d = json.loads(line)
            if d.get("kind") in ("dmma", "dmma_sustained"):
                best = max(best, float(d["tflops"]))
    except OSError:
        pass
    if best > 0:
        return best, "measured DMMA (profiles/r01_fp64_peak.jsonl)"
    return 148 * 1.965e9 * 128 / 1e12, "nominal 148 SMs x 128 flop/clk x 1.965 GHz"


#: BASELINE.json configs: name -> (n, numpy seed, distribution, b, diagonal shift)
CONFIGS = {
    "c1": (2048, 0, "uniform", 128, 0.0),
    "c2": (8192, 1, "uniform", 256, 0.0),
    "c2s": (8192, 1, "uniform", 256, 8192.0),
    "c3": (16384, 2, "normal", 256, 0.0),
    "c4": (32768, 3, "uniform", 256, 0.0),
    "c5": (65536, 4, "normal", 512, 0.0),
}


def config_matrix(name: str, n: int | None = None) -> np.ndarray:
    """The seeded BASELINE matrix (numpy default_rng(seed), row-major draw order), generated in row
    chunks (the same sequence as one call) so C5's 34 GB needs no second copy."""
    n0, seed, dist_name, _, shift = CONFIGS[name]
    n = n0 if n is None else n
    g = np.random.default_rng(seed)
    a = np.empty((n, n))
    rows = max(1, (1 << 27) // n)
    for r0 in range(0, n, rows):
        r1 = min(n, r0 + rows)
        a[r0:r1] = g.uniform(-1.0, 1.0, size=(r1 - r0, n)) if dist_name == "uniform" else g.standard_normal((r1 - r0, n))
    if shift:
        a[np.diag_indices(n)] += shift
    return a


def workload_name(args) -> str:
    n0, seed, dist_name, _, shift = CONFIGS[args.config]
    d = "U[-1,1)" if dist_name == "uniform" else "N(0,1)"
    sh = f" + {shift:g} I" if shift else ""
    return f"{args.config.upper()}: LUpp n={args.n} {d} numpy seed {seed}{sh}, b={args.b}, look-ahead {args.lookahead}"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int = 0):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


def load_traffic() -> tuple[float | None, str | None]:
    """DRAM bytes per launch of the trailing-update GEMM from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    try:
        d = json.load(open(path))
        return float(d["dram_bytes_per_launch"]), d.get("source")
    except (OSError, KeyError, ValueError):
        return None, None


def cpu_sample(n: int, b: int, threads: int | None = None, cfg: str = "c4"):
    """The oracle port (bitwise the reference's arithmetic, all host threads) on the first blocked
    step of the same matrix; GFLOP/s = that step's flops / wall time.  Also returns the step's final
    outputs (pivots [0, b) and factor rows [0, b)) for the bench's parity check."""
    import oracle

    cores = threads or os.cpu_count() or 1
    oracle.set_threads(cores)
    a = config_matrix(cfg, n)
    piv = np.zeros(n, dtype=np.int64)
    t0 = time.perf_counter()
    oracle.getrf_steps_inplace(a, b, 1, piv)
    dt = time.perf_counter() - t0
    fl = oracle.step_flops(n, n, b, 0)
    return ({"value": fl / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "port",
             "sample": f"first blocked step (panel {n}x{b} + laswp + trsm + {n - b}^2x{b} gemm) of the n={n} "
                       f"{cfg.upper()} matrix, {fl / 1e9:.1f} GFLOP in {dt:.2f} s, oracle/pflu_oracle.c -O3 OpenMP"},
            piv[:b].copy(), a[:b].copy())


REF_SLAB = 4096  # columns of the bounded CPU sample: the first blocked step of the config's left n x 4096 slab


def _import_reference():
    """The UNMODIFIED reference package installed in baseline/_ref (pip --target); its
    numba cache goes to /tmp, never into the tree.  Returns the module or None."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "panelforge")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/pflu_numba_cache")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import panelforge  # noqa: F401
    except Exception:  # noqa: BLE001  (numba missing etc.: reported as unavailable)
        return None
    return panelforge


def reference_step_sample(pf, pool, a: np.ndarray, b: int):
    """The reference's OWN code for the first blocked step of dmf_mtb / dmf_la (factor.py:396-411:
    _factor_panel + _update_columns with the full team) on the row-major n x slab array `a` (the
    config matrix's left columns).  Returns (seconds, flops, pivots[:b], rows[:b])."""
    from panelforge import CacheConfig, Kind, Matrix
    from panelforge import factor as F
    from panelforge.runtime import MalleableTeam

    import oracle

    n, slab = a.shape
    m = Matrix.from_array(a)                       # column-major copy, outside the timer (bench.py:125-138)
    piv = np.zeros(slab, dtype=np.int64)
    tau = np.zeros(slab)
    team = MalleableTeam(pool.t, max_size=pool.t) if pool.t > 1 else None
    t0 = time.perf_counter()
    pfac, _ = F._factor_panel(Kind.LU, m, 0, 0, b, piv, tau)
    F._update_columns(Kind.LU, m, pfac, b, slab, CacheConfig(b=b), pool=pool, team=team)
    dt = time.perf_counter() - t0
    out = np.ascontiguousarray(m.array)
    return dt, oracle.step_flops(n, slab, b, 0), piv[:b] - 1, out[:b]


def reference_cpu(args) -> dict | None:
    """cpu_baseline.reference_numba: the reference's own numba code timed on the host cores beside the
    C port -- the first-step sample above (and the port on the same sample, bitwise-compared), plus
    a full dmf_la factorization of C1.  None if the reference is not installed (baseline/_ref)."""
    pf = _import_reference()
    if pf is None:
        return None
    import oracle
    from panelforge import CacheConfig, Kind, Matrix, Pool

    cores = os.cpu_count() or 1
    with Pool(cores) as pool:
        warm = np.random.default_rng(0).uniform(-1, 1, (256, 256))
        pf.dmf_la(Matrix.from_array(warm), CacheConfig(b=64), pool, Kind.LU)   # numba warm-up (bench.py:125)
        slab = np.ascontiguousarray(config_matrix(args.config, args.n)[:, :REF_SLAB])
        dt, fl, rpiv, rrows = reference_step_sample(pf, pool, slab, args.b)
        a1 = config_matrix("c1")
        t0 = time.perf_counter()
        pf.dmf_la(Matrix.from_array(a1), CacheConfig(b=128), pool, Kind.LU)
        t_c1 = time.perf_counter() - t0
    oracle.set_threads(cores)
    port = slab
    ppiv = np.zeros(REF_SLAB, dtype=np.int64)
    t0 = time.perf_counter()
    oracle.getrf_steps_inplace(port, args.b, 1, ppiv)
    t_port = time.perf_counter() - t0
    return {"value": fl / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"reference panelforge (baseline/_ref, numba, Pool({cores})): first blocked step "
                      f"(_factor_panel + _update_columns) of the {args.config.upper()} matrix's left "
                      f"{args.n}x{REF_SLAB} slab, {fl / 1e9:.1f} GFLOP in {dt:.2f} s",
            "port_same_sample_gflops": fl / t_port / 1e9,
            "port_bitwise_equal_on_sample": bool(np.array_equal(rpiv, ppiv[:args.b]) and
                                                 rrows.tobytes() == port[:args.b].tobytes()),
            "c1_dmf_la_seconds": t_c1, "c1_dmf_la_gflops": lu_flops(2048) / t_c1 / 1e9}


def run_reference(args) -> None:
    """--impl reference: the reference's CPU implementation timed on the host cores, on bounded
    samples of the same workload.  With the reference installed (baseline/_ref) every step is ITS
    OWN code for the first blocked step of the config matrix's left n x 4096 slab (reference
    numba, Pool(all host threads)); otherwise the oracle port on the full first blocked step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pf = _import_reference()
    if pf is not None:
        run_reference_numba(args, pf)
        return
    import oracle

    n, b = args.n, args.b
    cores = os.cpu_count() or 1
    oracle.set_threads(cores)
    pristine = config_matrix(args.config, n)
    work = np.empty_like(pristine)
    piv = np.zeros(n, dtype=np.int64)
    fl = oracle.step_flops(n, n, b, 0)
    times = []
    for it in range(args.warmup + args.steps):
        np.copyto(work, pristine)
        t0 = time.perf_counter()
        oracle.getrf_steps_inplace(work, b, 1, piv)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = fl * len(times) / tot / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C4: LUpp n={n} U[-1,1) seed 3, b={b}, look-ahead 1",
                   "sample": "first blocked step of C4 per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"first blocked step of the n={n} {args.config.upper()} matrix ({fl / 1e9:.1f} GFLOP) per step; "
                                   "oracle/pflu_oracle.c is op-for-op the reference (pinned bitwise, tests/test_oracle.py)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def golden_parity(args, d_a0, d_lu, piv) -> dict:
    """Full-size parity of the timed run against the committed golden data (tests/golden/: the
    reference's own C1-C4 factors, the pinned oracle's C5): the FULL pivot vector (north_star's tie
    rule), plus one exact-mode factorization (reference rounding, outside the timed region) whose
    sha256 must equal the golden sha -- it is then the reference's factor, so max|LU - LU_exact| /
    ||A||_max is north_star's max|LU_gpu - LU_ref| / ||A||_max."""
    import hashlib

    import torch

    from paper_1804_07017_b200 import getrf_device

    gdir = os.path.join(ROOT, "tests", "golden")
    try:
        meta = json.load(open(os.path.join(gdir, "configs.json")))
        pivs = np.load(os.path.join(gdir, "configs_pivots.npz"))
        ties = np.load(os.path.join(gdir, "configs_ties.npz"))
    except OSError:
        return {"golden": "missing"}
    name = args.config
    n0, _, _, b0, _ = CONFIGS[name]
    if name not in meta or name not in pivs.files or args.n != n0 or args.b != b0:
        return {"golden": f"none for {name} at n={args.n} b={args.b}"}
    want = pivs[name].astype(np.int64)
    got = piv.cpu().numpy()
    diff = np.nonzero(got != want)[0]
    out = {"golden_source": meta[name].get("source", "reference"),
           "pivots_full_equal_golden": bool(len(diff) == 0),
           "pivots_first_mismatch": int(diff[0]) if len(diff) else None}
    if len(diff):
        t = ties[name] if name in ties.files else np.zeros((0, 4))
        row = t[t[:, 0] == diff[0]] if len(t) else t
        out["pivots_tie_rule_ok"] = bool(len(row) and (row[0, 1] - row[0, 2]) / row[0, 1] <= 1e-12
                                         and int(row[0, 3]) == int(got[diff[0]]))
    ex = d_a0.clone()
    piv_ex, _ = getrf_device(ex, args.b, args.lookahead, exact=True)
    torch.cuda.synchronize()
    h = hashlib.sha256()
    mx = 0.0
    for r0 in range(0, ex.shape[0], 4096):
        h.update(ex[r0:r0 + 4096].cpu().numpy().tobytes())
        mx = max(mx, float((d_lu[r0:r0 + 4096] - ex[r0:r0 + 4096]).abs().max()))
    amax = float(d_a0.abs().max())
    out["exact_sha256_equal_golden"] = h.hexdigest() == meta[name]["sha256_factors"]
    out["exact_pivots_equal_golden"] = bool(np.array_equal(piv_ex.cpu().numpy(), want))
    out["max_abs_lu_minus_ref_over_amax"] = mx / amax
    out["max_abs_bound"] = 10.0
    del ex
    torch.cuda.empty_cache()
    return out


def run_reference_numba(args, pf) -> None:
    from panelforge import CacheConfig, Kind, Matrix, Pool

    cores = os.cpu_count() or 1
    slab = np.ascontiguousarray(config_matrix(args.config, args.n)[:, :REF_SLAB])
    times, fl = [], 0.0
    with Pool(cores) as pool:
        warm = np.random.default_rng(0).uniform(-1, 1, (256, 256))
        pf.dmf_la(Matrix.from_array(warm), CacheConfig(b=64), pool, Kind.LU)
        for it in range(args.warmup + args.steps):
            dt, fl, _, _ = reference_step_sample(pf, pool, slab, args.b)
            if it >= args.warmup:
                times.append(dt)
    tot = sum(times)
    value = fl * len(times) / tot / 1e9
    sample = (f"reference panelforge (baseline/_ref, numba, Pool({cores})): first blocked step "
              f"(_factor_panel + _update_columns) of the {args.config.upper()} matrix's left {args.n}x{REF_SLAB} "
              f"slab ({fl / 1e9:.1f} GFLOP) per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args), "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_single(args) -> None:
    import torch

    from paper_1804_07017_b200 import _lib, getrf_device, lu_factor

    L = _lib.load()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    n, b, la = args.n, args.b, args.lookahead
    a_host = config_matrix(args.config, n)
    d_a0 = torch.from_numpy(a_host).to(dev)
    d_a = torch.empty_like(d_a0)
    piv = torch.empty(n, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    # The factorization is in place, so every step needs a pristine copy of the input.  Two work buffers:
    # while one is factored, the pristine matrix is copied back into the other on a side stream -- the copy
    # stays INSIDE the timed region (it competes for HBM with the factorization) but no longer serialises
    # with it.  When three copies of the matrix plus the parity block's buffers do not fit (C5), one buffer
    # and an in-step restore copy.
    free_b, _total_b = torch.cuda.mem_get_info(dev)
    double_buf = free_b > 3.2 * d_a0.numel() * 8
    d_b = torch.empty_like(d_a0) if double_buf else None
    bufs = [d_a, d_b] if double_buf else [d_a]
    s_restore = torch.cuda.Stream(device=dev) if double_buf else None
    ev_free = [torch.cuda.Event(), torch.cuda.Event()]   # buffer i: its factorization is done
    ev_ready = [torch.cuda.Event(), torch.cuda.Event()]  # buffer i: holds the pristine matrix again
    step_no = [0]
    if double_buf:
        d_a.copy_(d_a0)
        d_b.copy_(d_a0)
        for e in ev_ready:
            e.record(stream)

    def step(trace=None):
        if not double_buf:
            d_a.copy_(d_a0)
            _, info = getrf_device(d_a, b, la, piv=piv, trace=trace)
            return info
        i = step_no[0] & 1
        step_no[0] += 1
        stream.wait_event(ev_ready[i])
        _, info = getrf_device(bufs[i], b, la, piv=piv, trace=trace)
        ev_free[i].record(stream)
        with torch.cuda.stream(s_restore):  # restore this buffer while the next step factors the other one
            s_restore.wait_event(ev_free[i])
            bufs[i].copy_(d_a0, non_blocking=True)
            ev_ready[i].record(s_restore)
        return info

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    launches0 = L.pflu_launch_count()
    traces = []
    # the timed steps are traced for the roofline: only the GEMM and PF records (every record is two event
    # records on its stream; the TU_L / TU_R spans would add ~1% to the step)
    old_mask = L.pflu_set_trace_mask((1 << 4) | (1 << 0))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        tr = []
        step(trace=tr)
        traces.append(tr)
    if double_buf:  # the last restore copies belong to the timed region as well
        for e in ev_ready:
            stream.wait_event(e)
    e1.record(stream)
    torch.cuda.synchronize()
    launches = L.pflu_launch_count() - launches0
    clk = clocks.stop()
    L.pflu_set_trace_mask(old_mask)
    if double_buf:
        # both work buffers are pristine again: the parity block below checks one more (untimed) run of
        # the same call on the same input
        del d_b
        bufs = [d_a]
        torch.cuda.empty_cache()
        d_a.copy_(d_a0)
        getrf_device(d_a, b, la, piv=piv)
        torch.cuda.synchronize()
    total_ms = e0.elapsed_time(e1)
    ms_step = total_ms / args.steps
    value = lu_flops(n) / (ms_step * 1e-3) / 1e9

    # roofline of the dominant kernel: the trailing-update DMMA GEMM, from the live trace.  GEMM
    # launches of the column-chunk streams overlap in time, so the achieved rate is the GEMM flops
    # over the union of the intervals in which any trailing-update GEMM was running.
    g_flops, g_union_ms, g_cnt = 0.0, 0.0, 0
    for tr in traces:
        iv = []
        for ev in tr:
            if ev.label == "GEMM" and ev.flop > 0:
                g_flops += ev.flop
                g_cnt += 1
                iv.append((ev.start, ev.end))
        iv.sort()
        cur_s, cur_e = None, None
        for s_, e_ in iv:
            if cur_e is None or s_ > cur_e:
                if cur_e is not None:
                    g_union_ms += (cur_e - cur_s) * 1e3
                cur_s, cur_e = s_, e_
            else:
                cur_e = max(cur_e, e_)
        if cur_e is not None:
            g_union_ms += (cur_e - cur_s) * 1e3
    g_ms = g_union_ms
    peak, peak_src = fp64_peak()
    achieved = g_flops / (g_ms * 1e-3) / 1e12 if g_ms > 0 else None
    traffic, traffic_src = load_traffic()  # DRAM bytes of ONE launch at the step-0 shape (ncu --set full)
    pf_ms = sum((ev.end - ev.start) * 1e3 for ev in traces[-1] if ev.label == "PF")
    gemm_share = (g_ms / args.steps) / ms_step if ms_step else None

    # end to end through the public API with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if args.e2e_steps > 0:
        pinned = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        host = pinned.numpy()
        ts = []
        for it in range(args.e2e_steps + 1):
            np.copyto(host, a_host)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            lu, pv = lu_factor(host, b=b, lookahead=la)
            ts.append(time.perf_counter() - t0)
        ts = ts[1:]
        e2e = {"value": lu_flops(n) / statistics.mean(ts) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": n * n * 8, "d2h_bytes_per_step": n * n * 8 + n * 8,
               "api": "paper_1804_07017_b200.lu_factor(numpy pinned host array) -> pflu_getrf",
               "ms_per_step": 1e3 * statistics.mean(ts)}
        del pinned, host

    cpu = None
    parity = None
    if not args.no_cpu:
        cpu, ref_piv, ref_rows = cpu_sample(n, b, cfg=args.config)
        if not args.no_ref_cpu:
            cpu["reference_numba"] = reference_cpu(args)
    if not args.no_check:
        # parity of the timed call's output (the last timed step, or -- with two work buffers -- one more run
        # of it on the same input): the oracle's first blocked step (pivots and factor rows [0, b) are final
        # after it) and the full backward error on the GPU
        from paper_1804_07017_b200.cli import lu_residual_gpu

        parity = {"residual": lu_residual_gpu(d_a0, d_a, piv), "residual_bound": 10.0,
                  "residual_def": "||PA - LU||_F / (||A||_F n 2^-53), torch fp64 checker on the GPU"}
        parity.update(golden_parity(args, d_a0, d_a, piv))
        if not args.no_cpu:
            amax = float(np.max(np.abs(a_host)))
            parity["pivots_0_b_equal_oracle"] = bool(np.array_equal(piv[:b].cpu().numpy(), ref_piv))
            parity["rows_0_b_max_abs_diff_over_amax"] = float(np.max(np.abs(d_a[:b].cpu().numpy() - ref_rows))) / amax
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_name(args),
                   "n": n, "b": b, "lookahead": la, "parallelism": "single GPU",
                   "l2": ("inputs (%.1f GB) larger than L2; two work buffers: the pristine matrix is copied back into the idle "
                          "one on a side stream while the other is factored (the copies are inside the timed region)"
                          % (n * n * 8 / 1e9)) if double_buf else
                         ("inputs (%.1f GB) larger than L2; pristine matrix restored by a D2D copy inside each step"
                          % (n * n * 8 / 1e9)),
                   "fp64_peak_frac": value / 1e3 / peak},
        "roofline": {"bound": "tensor", "kernel": "gemm_dmma_ws<128x64x32, 2-stage TMA ring, producer warpgroup + 4 DMMA warps> (trailing update A22 -= L21*U12)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "peak_source": peak_src, "traffic_source": traffic_src,
                     "traffic_shape": "one launch at the step-0 shape 32512x32512x256 (algorithmic C r+w 16.9 GB)",
                     "launches_timed": g_cnt, "gemm_share_of_step": gemm_share,
                     "algorithmic": "2*M*N*b flop per TU_R chunk launch (M = n-(k+1)b rows, N = chunk columns >= (k+2)b); achieved = sum(flop) / union of GEMM-busy intervals"},
        "panel_ms_per_step": pf_ms,
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": launches,
        "cpu_baseline": cpu,
        "parity": parity,
    }
    print(json.dumps(line), flush=True)


def qr_flops(n: int) -> float:
    """4/3 n^3 (reference flops(Kind.QR), factor.py:208-215)."""
    return 4.0 * n ** 3 / 3.0


def run_single_qr(args) -> None:
    """--kind qr: the Householder QR path on the C4-shaped matrix: device-resident
    steps (restore + qr_factor on the torch stream) timed with CUDA events, e2e through
    qr_factor(pinned host array), CPU baseline = the oracle's first blocked QR step on the n x 4096
    left slab, parity = the timed run's reflector columns and R rows [0, b) vs that oracle step."""
    import torch

    import oracle
    from paper_1804_07017_b200 import _lib, qr_factor

    L = _lib.load()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    n, b, la = args.n, args.b, args.lookahead
    a_host = config_matrix(args.config, n)
    d_a0 = torch.from_numpy(a_host).to(dev)
    d_a = torch.empty_like(d_a0)
    stream = torch.cuda.current_stream(dev)

    def step():
        d_a.copy_(d_a0)
        return qr_factor(d_a, b=b, lookahead=la)[1]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    launches0 = L.pflu_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        tau = step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = L.pflu_launch_count() - launches0
    clk = clocks.stop()
    ms_step = e0.elapsed_time(e1) / args.steps
    value = qr_flops(n) / (ms_step * 1e-3) / 1e9
    peak, peak_src = fp64_peak()
    # roofline of the dominant work, the block-reflector GEMMs (W = V^T C, Z = T^T W, C -= V Z): one
    # extra TRACED factorization (single-stream schedule, not part of the timed steps); achieved =
    # 4 * m_p * n_c * b algorithmic flop per TU_R / TU_L record over the union of those intervals
    from paper_1804_07017_b200 import geqrf_device

    d_a.copy_(d_a0)
    tr = []
    geqrf_device(d_a, b, la, trace=tr)
    torch.cuda.synchronize()
    fl_tu, iv = 0.0, []
    for e in tr:
        if e.label in ("TU_R", "TU_L", "TU"):
            col0 = e.k * b
            mp = n - col0
            if e.label == "TU_L":
                nc = min(b, n - col0 - b)
            elif e.label == "TU_R":
                nc = n - col0 - b - min(b, n - col0 - b)
            else:
                nc = n - col0 - b
            fl_tu += 4.0 * mp * max(nc, 0) * min(b, n - col0)
            iv.append((e.start, e.end))
    iv.sort()
    busy, cs, ce = 0.0, None, None
    for s_, e_ in iv:
        if ce is None or s_ > ce:
            if ce is not None:
                busy += ce - cs
            cs, ce = s_, e_
        else:
            ce = max(ce, e_)
    if ce is not None:
        busy += ce - cs
    achieved = fl_tu / busy / 1e12 if busy > 0 else None
    roofline = {"bound": "tensor", "kernel": "block reflector: split-K gemm_dmma_t<128x64x32> (V^T C) + gemm_dmma_t (C -= V Z)",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": (achieved / peak) if achieved else None,
                "traffic": None, "peak_source": peak_src,
                "algorithmic": "4*m_p*n_c*b flop per TU_R / TU_L record (m_p = n - kb rows, n_c = updated columns) over the "
                               "union of their CUDA-event intervals, from one traced (single-stream) factorization"}
    e2e = None
    if args.e2e_steps > 0:
        pinned = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        host = pinned.numpy()
        ts = []
        for it in range(args.e2e_steps + 1):
            np.copyto(host, a_host)
            t0 = time.perf_counter()
            qr_factor(host, b=b, lookahead=la)
            ts.append(time.perf_counter() - t0)
        ts = ts[1:]
        e2e = {"value": qr_flops(n) / statistics.mean(ts) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": n * n * 8, "d2h_bytes_per_step": n * n * 8 + n * 8,
               "api": "paper_1804_07017_b200.qr_factor(numpy pinned host array) -> pflu_geqrf",
               "ms_per_step": 1e3 * statistics.mean(ts)}
        del pinned, host
    cpu, parity = None, None
    if not args.no_cpu:
        wcols = min(n, 4096)
        cores = os.cpu_count() or 1
        oracle.set_threads(cores)
        slab = np.ascontiguousarray(a_host[:, :wcols])
        t0 = time.perf_counter()
        ref, rtau = oracle.geqrf(slab, b, nsteps=1)
        dt = time.perf_counter() - t0
        fl = 2.0 * n * b * b + 4.0 * n * (wcols - b) * b
        cpu = {"value": fl / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"first blocked QR step (panel {n}x{b} qr_unb + larft + block reflector on {wcols - b} "
                         f"columns) of the n={n} C4 matrix's left {wcols} columns, {fl / 1e9:.1f} GFLOP in {dt:.2f} s"}
        got_v = d_a[:, :b].cpu().numpy()
        got_r = d_a[:b, :wcols].cpu().numpy()
        amax = float(np.max(np.abs(a_host)))
        parity = {"reflectors_0_b_max_abs_diff_over_amax": float(np.max(np.abs(got_v - ref[:, :b]))) / amax,
                  "r_rows_0_b_max_abs_diff_over_amax": float(np.max(np.abs(np.triu(got_r) - np.triu(ref[:b])))) / amax,
                  "tau_0_b_max_abs_diff": float(np.max(np.abs(tau[:b].cpu().numpy() - rtau[:b]))),
                  "bound": 1e-10}
    line = {
        "metric": "Householder QR FP64 GFLOP/s (4/3*n^3/t)", "value": value, "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"QR (Kind.QR) n={n} U[-1,1) numpy seed 3, b={b}, look-ahead {la}", "n": n, "b": b,
                   "lookahead": la, "parallelism": "single GPU", "fp64_peak_frac": value / 1e3 / peak,
                   "l2": "inputs (8.6 GB) larger than L2; pristine matrix restored by a D2D copy inside each step"},
        "roofline": roofline, "clocks": clk, "e2e": e2e, "gpu_launches": launches,
        "cpu_baseline": cpu, "parity": parity,
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(n_gpus: int) -> int:
    """`python bench.py --gpus N` outside torchrun: re-launch this command under
    torch.distributed.run with N ranks (one per GPU, rendezvous on 127.0.0.1); rank 0 prints the
    JSON line.  Fails loudly when fewer than N GPUs are visible (never silently measures fewer)."""
    selftest = "--selftest-launch" in sys.argv
    if not selftest:
        import torch

        have = torch.cuda.device_count()
        if have < n_gpus:
            print(f"bench.py: --gpus {n_gpus} requested but only {have} CUDA device(s) are visible", file=sys.stderr)
            return 2
    import socket

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # the communicator log (nranks) stays visible on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n_gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def selftest_launch(args) -> None:
    """--selftest-launch (CPU test of the launcher): every rank joins a gloo group and contributes
    one to an all-reduce; rank 0 prints the JSON line with n_gpus = the number of ranks that ran."""
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo")
    t = torch.ones(1)
    dist.all_reduce(t)
    if dist.get_rank() == 0:
        print(json.dumps({"metric": METRIC, "n_gpus": dist.get_world_size(), "ranks_seen": int(t.item()),
                          "selftest": True, "argv_gpus": args.gpus}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS),
                    help="BASELINE.json config (default C4, the one the metric's targets are quoted on)")
    ap.add_argument("--selftest-launch", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=None, help="override the config's n (same generator)")
    ap.add_argument("--b", type=int, default=None, help="override the config's block size")
    ap.add_argument("--lookahead", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the parity check of the timed run's output")
    ap.add_argument("--no-ref-cpu", action="store_true", help="skip timing the reference's own numba code")
    ap.add_argument("--dist", action="store_true", help="force the block-cyclic multi-GPU path (testing at N=1)")
    ap.add_argument("--kind", default="lu", choices=["lu", "qr"], help="qr: the Householder QR path (one GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    n0, _, _, b0, _ = CONFIGS[args.config]
    args.n = n0 if args.n is None else args.n
    args.b = b0 if args.b is None else args.b
    world = int(os.environ.get("WORLD_SIZE", "0") or 0)
    if args.gpus > 1 and world == 0 and args.impl == "ours":
        sys.exit(spawn_ranks(args.gpus))
    if world > 1 and args.gpus != world:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.selftest_launch:
        selftest_launch(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    if args.kind == "qr":
        run_single_qr(args)
        return
    if world > 1 or args.gpus > 1 or args.dist:
        from paper_1804_07017_b200.dist import bench_dist

        bench_dist(args, lu_flops, METRIC, UNIT, ClockSampler, fp64_peak, CONFIGS, workload_name(args))
        return
    run_single(args)


if __name__ == "__main__":
    main()
