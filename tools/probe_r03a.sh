set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_getrf.py -q -x -k "panel or recursive" > gpurun_out/p1_tests.log 2>&1; tail -3 gpurun_out/p1_tests.log
for K in 1 2 3; do timeout 120 python tools/panel_sweep.py --m 32768,16384,8192,4096,2048 --kernel $K --reps 5; done > gpurun_out/p1_sweep.log 2>&1
for LK in 1 2; do for LW in 16 32 64; do PFLU_REC_LEAFK=$LK PFLU_REC_LEAF=$LW timeout 120 python tools/panel_sweep.py --m 32768,8192,2048 --kernel 3 --reps 5 --tag "leafk=$LK leafw=$LW"; done; done >> gpurun_out/p1_sweep.log 2>&1
cat gpurun_out/p1_sweep.log | grep median
timeout 900 python tools/emu_scaling.py --ranks 1,2,4,8 > gpurun_out/p1_emu.log 2>&1
timeout 900 python tools/emu_scaling.py --ranks 2,8 --pf-kernel 3 >> gpurun_out/p1_emu.log 2>&1
cat gpurun_out/p1_emu.log
PFLU_PF_KERNEL=3 timeout 300 python bench.py --e2e-steps 0 --no-cpu > gpurun_out/p1_bench_rec.json 2>&1; tail -1 gpurun_out/p1_bench_rec.json | cut -c1-400
