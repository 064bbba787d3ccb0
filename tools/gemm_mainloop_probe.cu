// Upper bound of the GEMM mainloop: the production fragment loads (XOR-swizzled smem, 8 A + 4 B
// 64-bit LDS per k-quad) and 32 DMMAs per k-quad, but no cp.async and no barriers (smem contents
// stay fixed).  Variants: 2 CTAs x 4 warps per SM (production shape), 1 CTA x 8 warps.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

constexpr int BM = 128, BN = 64, BK = 16, ST = 4;

template <int WARPS, int MINB, bool BAR>
__global__ void __launch_bounds__(WARPS * 32, MINB) probe(double* out, int iters) {
  extern __shared__ double sm[];
  double* sA = sm;
  double* sB = sm + ST * BM * BK;
  for (int i = threadIdx.x; i < ST * (BM * BK + BK * BN); i += blockDim.x) sm[i] = 1.0 + i * 1e-12;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) & 3;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / 2, wn = warp % 2;
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
    const int kt = it & (ST - 1);
    if (BAR) __syncthreads();
    const double* cA = sA + kt * BM * BK;
    const double* cB = sB + kt * BK * BN;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = cA[(wm * 64 + i * 8 + g) * BK + ((kk + t) ^ ((g & 3) << 2))];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = -cB[(kk + t) * BN + ((wn * 32 + j * 8 + g) ^ (t << 2))];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 1.2345) out[0] = s;
}

template <int WARPS, int MINB, bool BAR>
void run(const char* name, double* out, int sms, int ctas_per_sm) {
  const int smem = ST * (BM * BK + BK * BN) * 8;
  cudaFuncSetAttribute(probe<WARPS, MINB, BAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<WARPS, MINB, BAR><<<sms * ctas_per_sm, WARPS * 32, smem>>>(out, 10);
  cudaEventRecord(e0);
  probe<WARPS, MINB, BAR><<<sms * ctas_per_sm, WARPS * 32, smem>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  // per warp per iteration: 4 k-quads x 32 DMMA x 512 flop
  double flops = 512.0 * 32 * 4 * (double)iters * WARPS * sms * ctas_per_sm;
  printf("%-44s %.2f TFLOP/s  (%s)\n", name, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, 2, false>("2 CTA/SM x 4 warps, smem LDS, no barrier", out, sms, 2);
  run<4, 2, true>("2 CTA/SM x 4 warps, smem LDS, barrier/stage", out, sms, 2);
  run<8, 1, false>("1 CTA/SM x 8 warps, smem LDS, no barrier", out, sms, 1);
  run<4, 1, false>("1 CTA/SM x 4 warps, smem LDS, no barrier", out, sms, 1);
  return 0;
}
