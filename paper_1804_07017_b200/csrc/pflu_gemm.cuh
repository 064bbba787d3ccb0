// pflu_gemm.cuh -- trailing-update GEMM on the FP64 tensor cores (DMMA), templated tiling.
//
// C(MxN) -= A(MxK) * B(KxN), row-major views into the matrix (the gemm(A22, A21, -A12) of
// _update_columns, factor.py:278-285 / kernels.py:173-218).  One DMMA.8x8x4 (mma.sync m8n8k4 f64)
// per 8x8 output block per k-quad; accumulators seeded from C (like macro_run, _jit.py:70-72); the
// B operand is negated by the instruction's operand modifier (exact), so the tensor core computes
// c + a * (-b) == c - a * b.  Operands stream through a multistage cp.async pipeline into
// XOR-swizzled shared tiles: A[m][k] at k ^ ((m & 3) << 2), B[k][n] at n ^ ((k & 3) << 2), which
// makes every 64-bit fragment load conflict free (two 128-byte wavefronts per warp).
#pragma once
#include "pflu_kernels.cuh"

namespace pflu {

template <int BM_, int BN_, int BK_, int ST_, int WM_, int WN_>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, ST = ST_, WM = WM_, WN = WN_;
  static constexpr int THREADS = WM * WN * 32;
  static constexpr int TM = BM / WM, TN = BN / WN;  // warp tile
  static constexpr int FM = TM / 8, FN = TN / 8;    // DMMA blocks per warp
  static constexpr int SMEM = ST * (BM * BK + BK * BN) * 8;
  static constexpr int MINB = (2 * SMEM <= 227 * 1024) ? 2 : 1;
  static_assert(BK % 16 == 0 && BN % 16 == 0 && TM % 8 == 0 && TN % 8 == 0, "tile shape");
};

template <class C, int VEC>
__device__ __forceinline__ void gemm_stage(const GemmArgs& p, double* sA, double* sB, int m0, int n0, int64_t k0,
                                           int tid) {
  if constexpr (VEC == 2) {
    constexpr int ACH = C::BK / 2, BCH = C::BN / 2;
#pragma unroll
    for (int i = 0; i < (C::BM * ACH + C::THREADS - 1) / C::THREADS; ++i) {
      const int q = tid + i * C::THREADS;
      if (q < C::BM * ACH) {
        const int row = q / ACH, k = (q % ACH) * 2;
        const int64_t gm = m0 + row, gk = k0 + k;
        const int bytes = gm < p.M ? (int)max((int64_t)0, min((int64_t)16, (p.K - gk) * 8)) : 0;
        const double* src = bytes ? p.a + gm * p.lda + gk : p.a;
        cp_async16(sA + row * C::BK + (k ^ ((row & 3) << 2)), src, bytes);
      }
    }
#pragma unroll
    for (int i = 0; i < (C::BK * BCH + C::THREADS - 1) / C::THREADS; ++i) {
      const int q = tid + i * C::THREADS;
      if (q < C::BK * BCH) {
        const int kr = q / BCH, n = (q % BCH) * 2;
        const int64_t gk = k0 + kr, gn = n0 + n;
        const int bytes = gk < p.K ? (int)max((int64_t)0, min((int64_t)16, (p.N - gn) * 8)) : 0;
        const double* src = bytes ? p.b + gk * p.ldb + gn : p.b;
        cp_async16(sB + kr * C::BN + (n ^ ((kr & 3) << 2)), src, bytes);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < (C::BM * C::BK + C::THREADS - 1) / C::THREADS; ++i) {
      const int q = tid + i * C::THREADS;
      if (q < C::BM * C::BK) {
        const int row = q / C::BK, k = q % C::BK;
        const int64_t gm = m0 + row, gk = k0 + k;
        const int bytes = (gm < p.M && gk < p.K) ? 8 : 0;
        const double* src = bytes ? p.a + gm * p.lda + gk : p.a;
        cp_async8(sA + row * C::BK + (k ^ ((row & 3) << 2)), src, bytes);
      }
    }
#pragma unroll
    for (int i = 0; i < (C::BK * C::BN + C::THREADS - 1) / C::THREADS; ++i) {
      const int q = tid + i * C::THREADS;
      if (q < C::BK * C::BN) {
        const int kr = q / C::BN, n = q % C::BN;
        const int64_t gk = k0 + kr, gn = n0 + n;
        const int bytes = (gk < p.K && gn < p.N) ? 8 : 0;
        const double* src = bytes ? p.b + gk * p.ldb + gn : p.b;
        cp_async8(sB + kr * C::BN + (n ^ ((kr & 3) << 2)), src, bytes);
      }
    }
  }
}

// Interior tiles (whole BM x BN tile inside C, whole K stage inside K): no predicates, per-thread
// source pointers and swizzled smem offsets computed once (row & 3 is invariant across a thread's
// chunks because chunk rows step by THREADS / chunks-per-row, a multiple of 4).
template <class C>
struct FastLoader {
  static constexpr int ACH = C::BK / 2, BCH = C::BN / 2;
  static constexpr int NA = C::BM * ACH / C::THREADS, NB = C::BK * BCH / C::THREADS;
  static constexpr int ASTEP = C::THREADS / ACH, BSTEP = C::THREADS / BCH;  // rows between chunks
  static_assert(C::BM * ACH % C::THREADS == 0 && C::BK * BCH % C::THREADS == 0, "even split");
  static_assert(ASTEP % 4 == 0 && BSTEP % 4 == 0, "swizzle phase must be invariant");
  const double* a0;
  const double* b0;
  int sa0, sb0;
  int64_t astride, bstride;
  __device__ __forceinline__ void init(const GemmArgs& p, int m0, int n0, int tid) {
    const int arow = tid / ACH, ak = (tid % ACH) * 2;
    const int brow = tid / BCH, bn = (tid % BCH) * 2;
    a0 = p.a + (int64_t)(m0 + arow) * p.lda + ak;
    b0 = p.b + (int64_t)brow * p.ldb + n0 + bn;
    sa0 = arow * C::BK + (ak ^ ((arow & 3) << 2));
    sb0 = brow * C::BN + (bn ^ ((brow & 3) << 2));
    astride = (int64_t)ASTEP * p.lda;
    bstride = (int64_t)BSTEP * p.ldb;
  }
  __device__ __forceinline__ void load(double* sA, double* sB, int64_t k0) const {
    const double* ap = a0 + k0;
#pragma unroll
    for (int i = 0; i < NA; ++i) cp_async16(sA + sa0 + i * ASTEP * C::BK, ap + i * astride, 16);
    const double* bp = b0 + k0 * (bstride / BSTEP);
#pragma unroll
    for (int i = 0; i < NB; ++i) cp_async16(sB + sb0 + i * BSTEP * C::BN, bp + i * bstride, 16);
  }
};

template <class C, int VEC>
__global__ void __launch_bounds__(C::THREADS, C::MINB) gemm_dmma_t(GemmArgs p) {
  extern __shared__ __align__(128) double gm_smem[];
  double* sA = gm_smem;
  double* sB = gm_smem + C::ST * C::BM * C::BK;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / C::WN, wn = warp % C::WN;
  int tm, tn;
  tile_coords(blockIdx.x, p.tiles_m, p.tiles_n, tm, tn);
  const int m0 = tm * C::BM, n0 = tn * C::BN;
  const int KT = (int)((p.K + C::BK - 1) / C::BK);
  const int KTF = (int)(p.K / C::BK);  // stages fully inside K
  const bool full = VEC == 2 && m0 + C::BM <= p.M && n0 + C::BN <= p.N;
  FastLoader<C> fl;
  if (full) fl.init(p, m0, n0, tid);
  auto stage = [&](int s, int kt) {
    double* dA = sA + s * C::BM * C::BK;
    double* dB = sB + s * C::BK * C::BN;
    if (full && kt < KTF) fl.load(dA, dB, (int64_t)kt * C::BK);
    else gemm_stage<C, VEC>(p, dA, dB, m0, n0, (int64_t)kt * C::BK, tid);
  };
#pragma unroll
  for (int s = 0; s < C::ST - 1; ++s) {
    if (s < KT) stage(s, s);
    cp_async_commit();
  }
  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i) {
    const int64_t row = m0 + wm * C::TM + i * 8 + g;
#pragma unroll
    for (int j = 0; j < C::FN; ++j) {
      const int64_t col = n0 + wn * C::TN + j * 8 + 2 * t;
      const double* cp = p.c + row * p.ldc + col;
      if (VEC == 2 && row < p.M && col + 1 < p.N) {
        const double2 v = *reinterpret_cast<const double2*>(cp);
        acc[i][j][0] = v.x;
        acc[i][j][1] = v.y;
      } else {
        acc[i][j][0] = (row < p.M && col < p.N) ? cp[0] : 0.0;
        acc[i][j][1] = (row < p.M && col + 1 < p.N) ? cp[1] : 0.0;
      }
    }
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<C::ST - 2>();
    __syncthreads();
    {
      const int nk = kt + C::ST - 1;
      const int s = nk % C::ST;
      if (nk < KT) stage(s, nk);
      cp_async_commit();
    }
    const double* cA = sA + (kt % C::ST) * C::BM * C::BK;
    const double* cB = sB + (kt % C::ST) * C::BK * C::BN;
#pragma unroll
    for (int kk = 0; kk < C::BK; kk += 4) {
      double af[C::FM], bf[C::FN];
#pragma unroll
      for (int i = 0; i < C::FM; ++i) {
        const int row = wm * C::TM + i * 8 + g;
        af[i] = cA[row * C::BK + ((kk + t) ^ ((g & 3) << 2))];
      }
#pragma unroll
      for (int j = 0; j < C::FN; ++j) {
        const int col = wn * C::TN + j * 8 + g;
        bf[j] = -cB[(kk + t) * C::BN + (col ^ (t << 2))];
      }
#pragma unroll
      for (int i = 0; i < C::FM; ++i)
#pragma unroll
        for (int j = 0; j < C::FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < C::FM; ++i) {
    const int64_t row = m0 + wm * C::TM + i * 8 + g;
    if (row >= p.M) continue;
#pragma unroll
    for (int j = 0; j < C::FN; ++j) {
      const int64_t col = n0 + wn * C::TN + j * 8 + 2 * t;
      double* cp = p.c + row * p.ldc + col;
      if (VEC == 2 && col + 1 < p.N) {
        *reinterpret_cast<double2*>(cp) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        if (col < p.N) cp[0] = acc[i][j][0];
        if (col + 1 < p.N) cp[1] = acc[i][j][1];
      }
    }
  }
}

// Persistent form: gridDim.x CTAs stride over the tiles; the operand pipeline runs continuously
// across tile boundaries (the first stages of tile t+1 are issued while tile t computes its last
// stages), which removes CTA launch gaps and hides the per-tile pipeline fill.
template <class C, int VEC, bool PREF = false>
__global__ void __launch_bounds__(C::THREADS, C::MINB) gemm_dmma_persistent(GemmArgs p) {
  extern __shared__ __align__(128) double gm_smem[];
  double* sA = gm_smem;
  double* sB = gm_smem + C::ST * C::BM * C::BK;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / C::WN, wn = warp % C::WN;
  const int ntiles = p.tiles_m * p.tiles_n;
  const int KT = (int)((p.K + C::BK - 1) / C::BK);
  const int KTF = (int)(p.K / C::BK);
  // producer cursor: (tile, kt) of the next stage to issue
  int pt = blockIdx.x, pk = 0;
  FastLoader<C> fl;
  bool pfull = false;
  int pm0 = 0, pn0 = 0;
  auto set_ptile = [&](int tile) {
    int tm, tn;
    tile_coords(tile, p.tiles_m, p.tiles_n, tm, tn);
    pm0 = tm * C::BM;
    pn0 = tn * C::BN;
    pfull = VEC == 2 && pm0 + C::BM <= p.M && pn0 + C::BN <= p.N;
    if (pfull) fl.init(p, pm0, pn0, tid);
  };
  if (pt < ntiles) set_ptile(pt);
  int gstage = 0;  // global stage counter (slot = gstage % ST)
  auto issue = [&]() {
    if (pt < ntiles) {
      const int s = gstage % C::ST;
      double* dA = sA + s * C::BM * C::BK;
      double* dB = sB + s * C::BK * C::BN;
      if (pfull && pk < KTF) fl.load(dA, dB, (int64_t)pk * C::BK);
      else gemm_stage<C, VEC>(p, dA, dB, pm0, pn0, (int64_t)pk * C::BK, tid);
      if (++pk == KT) {
        pk = 0;
        pt += gridDim.x;
        if (pt < ntiles) set_ptile(pt);
      }
    }
    cp_async_commit();
    ++gstage;
  };
#pragma unroll 1
  for (int s = 0; s < C::ST - 1; ++s) issue();
  int cstage = 0;  // consumer stage counter
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int tm, tn;
    tile_coords(tile, p.tiles_m, p.tiles_n, tm, tn);
    const int m0 = tm * C::BM, n0 = tn * C::BN;
    double acc[C::FM][C::FN][2];
#pragma unroll
    for (int i = 0; i < C::FM; ++i) {
      const int64_t row = m0 + wm * C::TM + i * 8 + g;
#pragma unroll
      for (int j = 0; j < C::FN; ++j) {
        const int64_t col = n0 + wn * C::TN + j * 8 + 2 * t;
        const double* cp = p.c + row * p.ldc + col;
        if (VEC == 2 && row < p.M && col + 1 < p.N) {
          const double2 v = *reinterpret_cast<const double2*>(cp);
          acc[i][j][0] = v.x;
          acc[i][j][1] = v.y;
        } else {
          acc[i][j][0] = (row < p.M && col < p.N) ? cp[0] : 0.0;
          acc[i][j][1] = (row < p.M && col + 1 < p.N) ? cp[1] : 0.0;
        }
      }
    }
    for (int kt = 0; kt < KT; ++kt, ++cstage) {
      cp_async_wait<C::ST - 2>();
      __syncthreads();
      issue();
      if (PREF && kt == KT / 2) {
        // pull the next tile's C block into L2 so its accumulator load does not wait on HBM
        const int nt = tile + gridDim.x;
        if (nt < ntiles) {
          int ntm, ntn;
          tile_coords(nt, p.tiles_m, p.tiles_n, ntm, ntn);
          const int nm0 = ntm * C::BM, nn0 = ntn * C::BN;
          for (int r = tid; r < C::BM; r += C::THREADS) {
            const int64_t row = nm0 + r;
            if (row < p.M) {
              const double* rp = p.c + row * p.ldc + nn0;
#pragma unroll
              for (int cl = 0; cl < C::BN * 8; cl += 128)
                if (nn0 + cl / 8 < p.N) asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + cl / 8));
            }
          }
        }
      }
      const double* cA = sA + (cstage % C::ST) * C::BM * C::BK;
      const double* cB = sB + (cstage % C::ST) * C::BK * C::BN;
#pragma unroll
      for (int kk = 0; kk < C::BK; kk += 4) {
        double af[C::FM], bf[C::FN];
#pragma unroll
        for (int i = 0; i < C::FM; ++i) {
          const int row = wm * C::TM + i * 8 + g;
          af[i] = cA[row * C::BK + ((kk + t) ^ ((g & 3) << 2))];
        }
#pragma unroll
        for (int j = 0; j < C::FN; ++j) {
          const int col = wn * C::TN + j * 8 + g;
          bf[j] = -cB[(kk + t) * C::BN + (col ^ (t << 2))];
        }
#pragma unroll
        for (int i = 0; i < C::FM; ++i)
#pragma unroll
          for (int j = 0; j < C::FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
#pragma unroll
    for (int i = 0; i < C::FM; ++i) {
      const int64_t row = m0 + wm * C::TM + i * 8 + g;
      if (row >= p.M) continue;
#pragma unroll
      for (int j = 0; j < C::FN; ++j) {
        const int64_t col = n0 + wn * C::TN + j * 8 + 2 * t;
        double* cp = p.c + row * p.ldc + col;
        if (VEC == 2 && col + 1 < p.N) {
          *reinterpret_cast<double2*>(cp) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else {
          if (col < p.N) cp[0] = acc[i][j][0];
          if (col + 1 < p.N) cp[1] = acc[i][j][1];
        }
      }
    }
  }
  cp_async_wait<0>();
}

// variants swept by tools/gemm_once.py (PFLU_GEMM_VARIANT); the production choice is GV6
// (K stage 32 double-buffered: 33.6 TFLOP/s at the C4 step-0 shape vs 32.4 for GV0)
using GV0 = GemmCfg<128, 64, 16, 4, 2, 2>;   // 4 warps of 64x32, 2 CTAs/SM
using GV1 = GemmCfg<128, 128, 16, 4, 2, 4>;  // 8 warps of 64x32
using GV2 = GemmCfg<128, 128, 32, 3, 2, 4>;  // 8 warps of 64x32, K stage 32
using GV3 = GemmCfg<128, 64, 16, 4, 4, 2>;   // 8 warps of 32x32
using GV4 = GemmCfg<128, 128, 16, 4, 4, 4>;  // 16 warps of 32x32
using GV5 = GemmCfg<256, 64, 16, 3, 4, 2>;   // 8 warps of 64x32, tall tile
using GV6 = GemmCfg<128, 64, 32, 2, 2, 2>;   // 4 warps of 64x32, K stage 32 double-buffered, 2 CTAs/SM
using GV7 = GemmCfg<64, 64, 32, 3, 2, 2>;    // 4 warps of 32x32, K stage 32, 2 CTAs/SM
using GV8 = GemmCfg<128, 64, 32, 2, 4, 2>;   // 8 warps of 32x32, K stage 32 double-buffered, 2 CTAs/SM

}  // namespace pflu
