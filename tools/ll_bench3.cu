// Replicates the panel kernel's per-column exchange to find what makes it slow.
// flags: 1 = publish 32 data words, 2 = CTA 0 publishes a diag record, 4 = read winner data,
//        8 = fenced grid sync every 32 columns, 16 = owner-of-p reads diag record
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void put2(unsigned long long* p, unsigned a, unsigned b, unsigned flag) {
  unsigned long long v0 = ((unsigned long long)flag << 32) | a, v1 = ((unsigned long long)flag << 32) | b;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(v0), "l"(v1) : "memory");
}
__device__ __forceinline__ bool try2(const unsigned long long* p, unsigned flag, unsigned& a, unsigned& b) {
  unsigned long long v0, v1;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v0), "=l"(v1) : "l"(p) : "memory");
  a = (unsigned)v0; b = (unsigned)v1;
  return (unsigned)(v0 >> 32) == flag && (unsigned)(v1 >> 32) == flag;
}

__global__ void ex(unsigned long long* ll, int iters, unsigned base, int flags, long long* gat) {
  const int S = gridDim.x, q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rec = 80;
  unsigned long long* sync_words = ll + 2 * (S + 1) * rec;
  __shared__ int s_win;
  __shared__ int red[8];
  for (int i = 0; i < iters; ++i) {
    const unsigned flag = base + i;
    unsigned long long* slots = ll + (size_t)(i & 1) * (S + 1) * rec;
    const int winner = (i * 7 + 3) % S;  // pseudo-random pivot owner
    __syncthreads();
    if (warp == 0) {
      unsigned long long* my = slots + (size_t)q * rec;
      if (flags & 1) put2(my + 16 + 2 * lane, lane, q, flag);
      if (lane == 0) { put2(my, q, 0, flag); put2(my + 2, q, 0, flag); }
    } else if (warp == 1 && (flags & 2) && q == 0) {
      put2(slots + (size_t)S * rec + 16 + 2 * lane, lane, 0, flag);
    }
    long long t0 = clock64();
    if (tid < S) {
      unsigned a, b, c, d;
      bool o0 = false, o1 = false;
      while (!(o0 && o1)) {
        if (!o0) o0 = try2(slots + (size_t)tid * rec, flag, a, b);
        if (!o1) o1 = try2(slots + (size_t)tid * rec + 2, flag, c, d);
      }
    }
    if (lane == 0) red[warp] = 1;
    __syncthreads();
    if (tid == 0 && q == 0 && i < 256) gat[i] = clock64() - t0;
    if ((flags & 4) && warp == 0) {
      unsigned a, b;
      while (!try2(slots + (size_t)winner * rec + 16 + 2 * lane, flag, a, b)) {}
    }
    if ((flags & 16) && warp == 1 && q == winner && q != 0) {
      unsigned a, b;
      while (!try2(slots + (size_t)S * rec + 16 + 2 * lane, flag, a, b)) {}
    }
    __syncthreads();
    if ((flags & 8) && (i % 32) == 31) {
      __syncthreads();
      if (tid == 0) { __threadfence(); put2(sync_words + 2 * q, 0, 0, flag); }
      if (tid < S) { unsigned a, b; while (!try2(sync_words + 2 * tid, flag, a, b)) {} }
      __threadfence();
      __syncthreads();
    }
  }
}

int main() {
  unsigned long long* w;
  long long *gat, h[256];
  cudaMalloc(&w, 1 << 22);
  cudaMemset(w, 0, 1 << 22);
  cudaMalloc(&gat, 256 * 8);
  unsigned base = 1;
  int S = 8;
  for (int flags : {0, 1, 3, 7, 15, 31, 8, 23}) {
    for (int rep = 0; rep < 2; ++rep) {
      int iters = 256;
      void* args[] = {&w, &iters, &base, &flags, &gat};
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)ex, dim3(S), dim3(256), args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      base += iters + 100;
      cudaMemcpy(h, gat, sizeof(h), cudaMemcpyDeviceToHost);
      if (rep) {
        printf("flags=%2d: %.3f us/iter; CTA0 gather us cols 30..45:", flags, ms * 1e3 / iters);
        for (int c = 30; c < 46; ++c) printf(" %.1f", h[c] / 1965.0);
        printf("  (%s)\n", cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
