# Round evidence pack (run under gpurun): bench line, ncu launch list of one factorization, panel and
# GEMM full captures.  Usage: bash tools/prof_round.sh r03
R=${1:-r03}
set -x
python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
tail -1 gpurun_out/bench_$R.json
L=$(python -c "import json;d=json.loads(open('gpurun_out/bench_$R.json').read().strip().splitlines()[-1]);print(d['gpu_launches']//d['steps'])")
echo "launches per step: $L"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3*L)) -c $L --csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu --no-check > gpurun_out/launches_$R.csv 2> gpurun_out/launches_$R.err
tail -2 gpurun_out/launches_$R.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:panel_kernel -s 3 -c 1 -o gpurun_out/panel_cl_full_$R python tools/panel_once.py 32768 256 > gpurun_out/ncu_panel_full.log 2>&1
tail -2 gpurun_out/ncu_panel_full.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_dmma -s 2 -c 1 -o gpurun_out/gemm_full_$R python tools/gemm_once.py 32512 32512 256 1 > gpurun_out/ncu_gemm_full.log 2>&1
tail -2 gpurun_out/ncu_gemm_full.log
# TRSM (FP64 pipe) and laswp (HBM) evidence: one launch each, tools/swap_dmma_once.py
timeout 600 ncu --set full --import-source on --clock-control none -k regex:swap_trsm_dmma -s 2 -c 1 -o gpurun_out/trsm_full_$R python tools/swap_dmma_once.py > gpurun_out/ncu_trsm_full.log 2>&1
tail -2 gpurun_out/ncu_trsm_full.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:swap_trsm_kernel -s 2 -c 1 -o gpurun_out/lswap_full_$R python tools/swap_dmma_once.py > gpurun_out/ncu_lswap_full.log 2>&1
tail -2 gpurun_out/ncu_lswap_full.log
