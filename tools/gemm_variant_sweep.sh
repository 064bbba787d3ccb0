# Every trailing-GEMM variant at the C4 step-0 shape and a mid shape (under gpurun).
for V in 0 1 2 3 4 5 6 7 8 10 13 16 17 20 21 40; do
  for S in "32512 32512 256" "16384 16384 256"; do
    echo -n "variant $V: "; PFLU_GEMM_VARIANT=$V timeout 60 python tools/gemm_once.py $S 5 2>&1 | tail -1
  done
done
echo -n "tma: "; PFLU_GEMM_TMA=1 timeout 60 python tools/gemm_once.py 32512 32512 256 5 cublas 2>&1 | tail -2
