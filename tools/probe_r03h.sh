PFLU_GEMM_TMA=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" > gpurun_out/p8_tests.log 2>&1; tail -2 gpurun_out/p8_tests.log
for T in 1 0; do for S in "32512 32512 256" "16384 16384 256" "8192 8192 256" "32512 32512 512"; do PFLU_GEMM_TMA=$T timeout 60 python tools/gemm_once.py $S 10; done; done 2>&1 | tee gpurun_out/p8_gemm.log
PFLU_GEMM_TMA=1 timeout 300 python bench.py --e2e-steps 0 --no-cpu > gpurun_out/p8_bench.json 2>&1; tail -1 gpurun_out/p8_bench.json | cut -c1-250
