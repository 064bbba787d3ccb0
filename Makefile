# In-tree build of libpflu.so (sm_100a) and the CPU oracle; __graft_entry__.build() does the same.
NVCC ?= /usr/local/cuda/bin/nvcc
NVFLAGS = -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -std=c++17 --shared -Xcompiler -fPIC -ldl
SRC = paper_1804_07017_b200/csrc/pflu.cu
HDR = paper_1804_07017_b200/csrc/pflu_mg.cuh paper_1804_07017_b200/csrc/pflu_kernels.cuh paper_1804_07017_b200/csrc/pflu_panel.cuh paper_1804_07017_b200/csrc/pflu_gemm.cuh paper_1804_07017_b200/csrc/pflu_qr.cuh include/pflu.h

all: paper_1804_07017_b200/libpflu.so oracle/liboracle.so

paper_1804_07017_b200/libpflu.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -o $@ $(SRC)

oracle/liboracle.so: oracle/pflu_oracle.c
	$(MAKE) -s -C oracle

regs: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -o /tmp/pflu_regs.so $(SRC) 2>&1 | grep -E "Compiling|registers|spill"

.PHONY: all regs
