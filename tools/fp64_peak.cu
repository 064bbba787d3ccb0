// FP64 peak microbenchmark: DMMA (mma.sync m8n8k4 f64) vs DFMA, all SMs.
// Used once to calibrate the FP64 roofline denominator (MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 123.456) out[0] = s;
}

// numerics probe: one m8n8k4 with chosen operands vs sequential fma / mul+add
__global__ void dmma_probe(const double* A, const double* B, const double* C, double* D) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a = A[g * 4 + t];      // A 8x4 row-major
  double b = B[t * 8 + g];      // B 4x8 row-major, fragment B[t][g]
  double d0 = C[g * 8 + 2 * t], d1 = C[g * 8 + 2 * t + 1];
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  D[g * 8 + 2 * t] = d0; D[g * 8 + 2 * t + 1] = d1;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%zu,\"clock_khz\":%d,\"regs_per_sm\":%d,\"coop\":%d}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, clk,
         p.regsPerMultiprocessor, p.cooperativeLaunch);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 2; ++rep) {
    for (int bpm : {1, 2, 4}) {
      for (int thr : {128, 256, 512}) {
        int iters = 20000;
        dmma_loop<<<sms * bpm, thr>>>(out, 100);
        cudaEventRecord(e0);
        dmma_loop<<<sms * bpm, thr>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 256 * 8 * (double)iters * (sms * bpm) * (thr / 32);
        printf("{\"kind\":\"dmma\",\"blocks_per_sm\":%d,\"threads\":%d,\"tflops\":%.2f,\"ms\":%.3f}\n", bpm, thr, flops / ms / 1e9, ms);
      }
    }
    for (int bpm : {1, 2, 4}) {
      int thr = 512, iters = 20000;
      dfma_loop<<<sms * bpm, thr>>>(out, 100);
      cudaEventRecord(e0);
      dfma_loop<<<sms * bpm, thr>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16 * (double)iters * (sms * bpm) * thr;
      printf("{\"kind\":\"dfma\",\"blocks_per_sm\":%d,\"threads\":%d,\"tflops\":%.2f,\"ms\":%.3f}\n", bpm, thr, flops / ms / 1e9, ms);
    }
  }
  // sustained: DMMA for ~3 s
  {
    int iters = 200000; int bpm = 2, thr = 256;
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) dmma_loop<<<sms * bpm, thr>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 5 * 2.0 * 256 * 8 * (double)iters * (sms * bpm) * (thr / 32);
    printf("{\"kind\":\"dmma_sustained\",\"tflops\":%.2f,\"ms\":%.1f}\n", flops / ms / 1e9, ms);
  }
  // numerics probe
  double hA[32], hB[32], hC[64], hD[64];
  for (int i = 0; i < 32; ++i) { hA[i] = 1.0 + i * 0x1p-30; hB[i] = 1.0 - i * 0x1p-29; }
  for (int i = 0; i < 64; ++i) hC[i] = -4.0 + i * 0x1p-40;
  hA[0] = 1.0; hB[0] = 0x1p-53; hA[1] = 1.0; hB[8] = 0x1p-53; hC[0] = 1.0;  // tiny terms
  double *dA, *dB, *dC, *dD; cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512); cudaMalloc(&dD, 512);
  cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, hC, 512, cudaMemcpyHostToDevice);
  dmma_probe<<<1, 32>>>(dA, dB, dC, dD);
  cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
  int same_fma = 0, same_muladd = 0;
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 8; ++j) {
    double f = hC[i * 8 + j], m = hC[i * 8 + j];
    for (int k = 0; k < 4; ++k) { f = __builtin_fma(hA[i * 4 + k], hB[k * 8 + j], f); volatile double pr = hA[i * 4 + k] * hB[k * 8 + j]; m = m + pr; }
    same_fma += (f == hD[i * 8 + j]); same_muladd += (m == hD[i * 8 + j]);
  }
  printf("{\"probe\":\"dmma_vs_seq\",\"same_as_fma_chain\":%d,\"same_as_mul_add\":%d,\"of\":64,\"d00\":%.17g}\n", same_fma, same_muladd, hD[0]);
  printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
