// All-to-all flag exchange latency between S co-resident CTAs (LL words): layouts and protocols.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void put(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long get(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// mode 0: all-to-all, slot stride `stride` words; mode 1: leader gathers, broadcasts one word;
// mode 2: all-to-all with nanosleep backoff
template <int MODE>
__global__ void a2a(unsigned long long* words, int iters, unsigned base, int stride, long long* out,
                    unsigned long long* check) {
  const int S = gridDim.x, q = blockIdx.x, tid = threadIdx.x;
  __shared__ unsigned long long sum;
  long long t0 = clock64();
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
    const unsigned long long flag = base + i;
    unsigned long long* slot = words + (size_t)(i & 1) * (256 * 32 + 64);
    if (tid == 0) sum = 0;
    __syncthreads();
    if (tid == 0) put(slot + q * stride, (flag << 32) | (unsigned)(q + i));
    if (MODE == 1) {
      unsigned long long* res = slot + 256 * 32;
      if (q == 0) {
        unsigned long long v = 0;
        if (tid < S) {
          do { v = get(slot + tid * stride); } while ((v >> 32) != flag);
          atomicAdd(&sum, v & 0xffffffffull);
        }
        __syncthreads();
        if (tid == 0) put(res, (flag << 32) | (unsigned)sum);
      }
      if (tid == 0) {
        unsigned long long v;
        do { v = get(res); } while ((v >> 32) != flag);
        acc += v & 0xffffffffull;
      }
    } else {
      if (tid < S) {
        unsigned long long v;
        int spins = 0;
        do {
          v = get(slot + tid * stride);
          if (MODE == 2 && (v >> 32) != flag && ++spins > 2) __nanosleep(32);
        } while ((v >> 32) != flag);
        atomicAdd(&sum, v & 0xffffffffull);
      }
      __syncthreads();
      if (tid == 0) acc += sum;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) { out[q] = t1 - t0; check[q] = acc; }
}

int main() {
  unsigned long long *w, *chk;
  long long* out;
  cudaMalloc(&w, 1 << 22);
  cudaMemset(w, 0, 1 << 22);
  cudaMalloc(&out, 4096 * 8);
  cudaMalloc(&chk, 4096 * 8);
  unsigned base = 1;
  for (int S : {8, 32, 64, 148}) {
    struct { int mode, stride; const char* name; } cfgs[] = {
        {0, 4, "a2a stride 32B"}, {0, 16, "a2a stride 128B"}, {0, 32, "a2a stride 256B"},
        {1, 16, "leader 2-hop 128B"}, {2, 16, "a2a 128B nanosleep"}};
    for (auto& cf : cfgs) {
      int iters = 2000;
      void (*k)(unsigned long long*, int, unsigned, int, long long*, unsigned long long*) =
          cf.mode == 0 ? a2a<0> : cf.mode == 1 ? a2a<1> : a2a<2>;
      int stride = cf.stride;
      void* args[] = {&w, &iters, &base, &stride, &out, &chk};
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)k, dim3(S), dim3(256), args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long h[2];
      cudaMemcpy(h, chk, 16, cudaMemcpyDeviceToHost);
      // expected per-iteration sum = sum_q (q + i) = S(S-1)/2 + S*i
      unsigned long long exp = 0;
      for (int i = 0; i < iters; ++i) exp += (unsigned long long)S * (S - 1) / 2 + (unsigned long long)S * i;
      base += iters + 10;
      printf("S=%3d %-22s %.3f us/exchange  check=%s  err=%s\n", S, cf.name, ms * 1e3 / iters,
             (h[0] == exp && h[1] == exp) ? "ok" : "BAD", cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
