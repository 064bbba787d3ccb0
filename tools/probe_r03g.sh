PFLU_GEMM_TMA=1 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_getrf.py -q -x -k "gemm or small_dmma or c1_dmma or c2" > gpurun_out/p7_tests.log 2>&1; tail -3 gpurun_out/p7_tests.log
for T in 1 0; do for S in "32512 32512 256" "16384 16384 256" "8192 8192 256" "32512 32512 512"; do PFLU_GEMM_TMA=$T timeout 60 python tools/gemm_once.py $S 10; done; done 2>&1 | tee gpurun_out/p7_gemm.log
PFLU_GEMM_TMA=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_dmma -s 2 -c 1 -o gpurun_out/gemm_tma64_full python tools/gemm_once.py 16384 16384 256 3 > gpurun_out/p7_ncu1.log 2>&1
PFLU_GEMM_TMA=1 timeout 300 python bench.py --e2e-steps 0 --no-cpu > gpurun_out/p7_bench.json 2>&1; tail -1 gpurun_out/p7_bench.json | cut -c1-250
