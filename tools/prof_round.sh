set -x
python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
tail -1 gpurun_out/bench_r02.json
L=$(python -c "import json;d=json.loads(open('gpurun_out/bench_r02.json').read().strip().splitlines()[-1]);print(d['gpu_launches']//d['steps'])")
echo "launches per step: $L"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3*L)) -c $L --csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/launches_r02.csv 2> gpurun_out/launches_r02.err
tail -2 gpurun_out/launches_r02.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:panel_kernel -s 3 -c 1 -o gpurun_out/panel_cl_full_r02 python tools/panel_once.py 32768 256 > gpurun_out/ncu_panel_full.log 2>&1
tail -2 gpurun_out/ncu_panel_full.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_dmma -s 2 -c 1 -o gpurun_out/gemm_full_r02 python tools/gemm_once.py 32512 32512 256 1 > gpurun_out/ncu_gemm_full.log 2>&1
tail -2 gpurun_out/ncu_gemm_full.log
