set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_getrf.py -q -x -k "not c4 and not c5" > gpurun_out/p4_tests.log 2>&1; tail -3 gpurun_out/p4_tests.log
timeout 120 python tools/panel_sweep.py --m 32768,16384,8192,4096,2048,1024 --kernel 2 --reps 5 > gpurun_out/p4_sweep.log 2>&1
timeout 120 python tools/panel_sweep.py --m 4096,2048,1024 --w 128 --kernel 2 --reps 5 >> gpurun_out/p4_sweep.log 2>&1
grep median gpurun_out/p4_sweep.log
for M in 2048 8192; do timeout 60 python tools/panel_prof.py $M 256 0 0 0 2; done > gpurun_out/p4_prof.log 2>&1
cat gpurun_out/p4_prof.log
