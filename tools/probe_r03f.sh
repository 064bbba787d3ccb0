set -x
PFLU_GEMM_TMA=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_dmma -s 2 -c 1 -o gpurun_out/gemm_tma_full python tools/gemm_once.py 16384 16384 256 3 > gpurun_out/p6_ncu1.log 2>&1
PFLU_GEMM_TMA=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_dmma -s 2 -c 1 -o gpurun_out/gemm_cpa_full python tools/gemm_once.py 16384 16384 256 3 > gpurun_out/p6_ncu2.log 2>&1
tail -2 gpurun_out/p6_ncu1.log gpurun_out/p6_ncu2.log
