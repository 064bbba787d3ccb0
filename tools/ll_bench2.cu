// Exchange latency: scalar vs v2 relaxed LL words, record stride as in the panel kernel.
#include <cstdio>
#include <cuda_runtime.h>

template <int V2>
__global__ void a2a(unsigned long long* words, int iters, unsigned base, int stride) {
  const int S = gridDim.x, q = blockIdx.x, tid = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    const unsigned long long flag = base + i;
    unsigned long long* slot = words + (size_t)(i & 1) * (256 * stride);
    if (tid == 0) {
      unsigned long long v = (flag << 32) | (unsigned)q;
      if (V2) asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(slot + q * stride), "l"(v), "l"(v) : "memory");
      else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(slot + q * stride), "l"(v) : "memory");
    }
    if (tid < S) {
      unsigned long long v0, v1;
      do {
        if (V2) asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v0), "=l"(v1) : "l"(slot + tid * stride) : "memory");
        else { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v0) : "l"(slot + tid * stride) : "memory"); v1 = v0; }
      } while ((v0 >> 32) != flag || (v1 >> 32) != flag);
    }
    __syncthreads();
  }
}

int main() {
  unsigned long long* w;
  cudaMalloc(&w, 1 << 24);
  cudaMemset(w, 0, 1 << 24);
  unsigned base = 1;
  for (int rep = 0; rep < 2; ++rep)
  for (int S : {8, 32, 148}) {
    for (int v2 = 0; v2 < 2; ++v2) for (int stride : {16, 80}) {
      int iters = 4000;
      void* args[] = {&w, &iters, &base, &stride};
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel(v2 ? (void*)a2a<1> : (void*)a2a<0>, dim3(S), dim3(256), args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      base += iters + 10;
      if (rep) printf("S=%3d %s stride=%d words: %.3f us/exchange (%s)\n", S, v2 ? "v2    " : "scalar", stride, ms * 1e3 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
