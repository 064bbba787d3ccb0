"""Summarise QR ncu evidence (run here on the .ncu-rep / csv files gpurun brought back):
per-kernel share of one factorization's launch list, plus key counters of the full captures."""
import collections
import csv
import io
import json
import re
import subprocess
import sys

launches, leaf_rep, gemm_rep, out = sys.argv[1:5]
rows = list(csv.reader(open(launches)))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    name = re.sub(r"\(.*", "", r[ki])[:90]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
tot = sum(v[1] for v in agg.values())
share = [{"kernel": k, "launches": c, "ms": round(t, 3), "share": round(t / tot, 4)}
         for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])]

want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__shared_mem_per_block_dynamic"]


def counters(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hd, un, va = rr[0], rr[1], rr[2]
    d = {k: f"{va[hd.index(k)]} {un[hd.index(k)]}".strip() for k in want if k in hd}
    d["kernel"] = va[hd.index("Kernel Name")] if "Kernel Name" in hd else None
    return d


res = {"source": "ncu --metrics gpu__time_duration.sum --clock-control none (launch list, one n=8192 b=256 "
                 "look-ahead-1 QR, serialised/cold) and ncu --set full --clock-control none captures",
       "launch_list_total_ms": round(tot, 3), "per_kernel": share,
       "leaf_kernel_full": counters(leaf_rep), "split_gemm_full": counters(gemm_rep)}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1)[:3000])
