timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r03_pytest_gpu.log 2>&1; tail -3 gpurun_out/r03_pytest_gpu.log
timeout 600 python bench.py --dist --steps 2 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/r03_bench_dist1.json 2> gpurun_out/r03_bench_dist1.err; tail -1 gpurun_out/r03_bench_dist1.json | cut -c1-300; tail -3 gpurun_out/r03_bench_dist1.err
bash tools/prof_round.sh r03 > gpurun_out/r03_prof.log 2>&1; tail -12 gpurun_out/r03_prof.log
