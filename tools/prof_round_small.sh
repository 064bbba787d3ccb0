# Round evidence (small enough to come back through gpurun): bench line, launch list of one C4
# factorization summarised on the box, GEMM full capture summarised on the box.  Usage: bash tools/prof_round_small.sh r04
R=${1:-r04}
set -x
python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
L=$(python -c "import json;d=json.loads(open('gpurun_out/bench_$R.json').read().strip().splitlines()[-1]);print(d['gpu_launches']//d['steps'])")
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3*L)) -c $L --csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu --no-check > gpurun_out/launches_$R.csv 2> gpurun_out/launches_$R.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_dmma -s 2 -c 1 -o /tmp/gemm_full_$R python tools/gemm_once.py 32512 32512 256 1 > gpurun_out/ncu_gemm_full.log 2>&1
python tools/ncu_gemm_summary.py /tmp/gemm_full_$R.ncu-rep gpurun_out/${R}_gemm_full_summary.json gemm_dmma 32512x32512x256 > gpurun_out/gemm_summary.log 2>&1
ls -la gpurun_out
