"""Summarise an `ncu --set full` capture of one trailing-update GEMM launch into the JSON that
bench.py reads for roofline.traffic (profiles/gemm_traffic.json) -- run here, on the .ncu-rep."""
import csv
import io
import json
import subprocess
import sys

rep, out, kernel, shape = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
M, N, K = (int(x) for x in shape.split("x"))
raw = open(rep).read() if rep.endswith(".csv") else \
    subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
raw = raw[raw.index('"ID"'):] if '"ID"' in raw else raw
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__grid_size",
        "launch__registers_per_thread", "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]
m = {k: f"{vals[hdr.index(k)]} {units[hdr.index(k)]}" for k in want if k in hdr}


def to_bytes(s):
    v, u = s.split()
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


def to_s(s):
    v, u = s.split()
    return float(v.replace(",", "")) * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6,
                                         "ms": 1e-3, "second": 1.0}[u]


dram = to_bytes(m["dram__bytes_read.sum"]) + to_bytes(m["dram__bytes_write.sum"])
dur = to_s(m["gpu__time_duration.sum"])
d = {"source": f"ncu --set full --clock-control none, {out} (tools/gemm_once.py {M} {N} {K} 1, one launch of {kernel})",
     "kernel": kernel, "M": M, "N": N, "K": K, "dram_bytes_per_launch": dram,
     "algorithmic_bytes_C_rw": 2 * M * N * 8, "duration_s": dur, "tflops_under_ncu": 2 * M * N * K / dur / 1e12,
     "metrics": m}
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d, indent=1))
