# QR evidence under gpurun: bench line (--kind qr), launch list of one n=8192 QR, full capture of
# one leaf kernel (32768-row panel) and of one split-K GEMM.
set -x
timeout 900 python bench.py --kind qr --steps 3 --warmup 3 > gpurun_out/qr_bench_line.json 2> gpurun_out/qr_bench.err
python tools/qr_once.py 8192 256 1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qr_launches_8192.csv \
      python tools/qr_once.py 8192 256 1 > gpurun_out/qr_ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:qr_leaf_kernel --launch-skip 8 -c 1 \
    -o gpurun_out/qr_leaf_full -f python tools/qr_once.py 32768 256 0 > gpurun_out/qr_ncu_leaf.log 2>&1
ncu --set full --clock-control none -k regex:gemm_dmma_t --launch-skip 40 -c 1 \
    -o gpurun_out/qr_gemm_full -f python tools/qr_once.py 16384 256 0 > gpurun_out/qr_ncu_gemm.log 2>&1
ls -la gpurun_out
