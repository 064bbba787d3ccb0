timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "panel" > gpurun_out/p11_tests.log 2>&1; tail -2 gpurun_out/p11_tests.log
timeout 120 python tools/panel_sweep.py --m 32768,16384,8192,4096,2048 --kernel 1,2 --reps 5 > gpurun_out/p11_sweep.log 2>&1; grep median gpurun_out/p11_sweep.log
timeout 300 python bench.py --e2e-steps 0 --no-cpu --no-check 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['achieved'], d['panel_ms_per_step'])"
