# Round evidence pack (run under gpurun): bench line, ncu launch list of one factorization, GEMM /
# panel / TRSM / laswp full captures.  The .ncu-rep files stay on the box (/tmp/prof); their raw
# pages come back as CSV (gpurun_out/ is capped at 64 MiB).  Usage: bash tools/prof_round.sh r05
R=${1:-r06}
P=/tmp/prof; mkdir -p $P gpurun_out
set -x
python bench.py --e2e-steps 1 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
tail -1 gpurun_out/bench_$R.json
L=$(python -c "import json;d=json.loads(open('gpurun_out/bench_$R.json').read().strip().splitlines()[-1]);print(d['gpu_launches']//d['steps'])")
echo "launches per step: $L"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3*L)) -c $L --csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu --no-check > gpurun_out/launches_$R.csv 2> gpurun_out/launches_$R.err
tail -2 gpurun_out/launches_$R.err
cap() {  # name kernel-regex command...
  local name=$1 rx=$2; shift 2
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$rx -s 2 -c 1 -o $P/${name}_$R "$@" > gpurun_out/ncu_${name}_$R.log 2>&1
  tail -2 gpurun_out/ncu_${name}_$R.log
  ncu -i $P/${name}_$R.ncu-rep --page raw --csv > gpurun_out/${name}_${R}_raw.csv 2>/dev/null
  ncu -i $P/${name}_$R.ncu-rep --page source --csv 2>/dev/null | head -c 8000000 > gpurun_out/${name}_${R}_source.csv
}
cap gemm gemm_dmma python tools/gemm_once.py 32512 32512 256 1
cap panel panel_kernel python tools/panel_once.py 2048 256 0 0 2     # v2 cluster leaf (no top-level split below 4096 rows)
cap panelmc panel_kernel python tools/panel_once.py 32768 128 0 0 4  # multi-cluster kernel, one 128-column half
cap trsm swap_trsm_dmma python tools/swap_dmma_once.py
cap lswap swap_trsm_kernel python tools/swap_dmma_once.py
