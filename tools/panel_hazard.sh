#!/bin/bash
# Re-check of the panel kernel's codegen-sensitive zero-pivot failure: the
# production build compiles the exact flag into panel_kernel (the specialisation that once returned
# wrong pivots on the singular golden case); this also builds the round-1 runtime-flag variant
# (-DPFLU_PANEL_EXACT_RUNTIME) and runs the small golden cases and the zero-pivot stress against
# it, PFLU_STRESS_REPEATS times each.  GPU box.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=paper_1804_07017_b200/libpflu_ext.so
/usr/local/cuda/bin/nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -std=c++17 --shared -Xcompiler -fPIC \
  -DPFLU_PANEL_EXACT_RUNTIME -o $OUT paper_1804_07017_b200/csrc/pflu.cu || exit 1
export PFLU_LIB_PATH=$PWD/$OUT
export PFLU_STRESS_REPEATS=${PFLU_STRESS_REPEATS:-50}
python -m pytest tests/test_gpu_getrf.py -q -m gpu -k "small_golden_exact" -x 2>&1 | tail -3
python -m pytest tests/test_gpu_panel_stress.py -q -m gpu -x 2>&1 | tail -15
