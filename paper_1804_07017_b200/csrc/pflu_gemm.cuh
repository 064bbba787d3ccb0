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
#include <cuda.h>

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

// SPLIT (QR's tall-skinny products V^T C): blockIdx.y selects a K slice of p.kslice columns of A /
// rows of B and its own output slice p.c + blockIdx.y * p.cslice; accumulators start from zero, so
// slice s holds -(A_s B_s) and the caller sums the slices in a fixed order (deterministic).
template <class C, int VEC, bool SPLIT = false>
__global__ void __launch_bounds__(C::THREADS, C::MINB) gemm_dmma_t(GemmArgs p) {
  if constexpr (SPLIT) {
    const int64_t ks = (int64_t)blockIdx.y * p.kslice;
    p.a += ks;
    p.b += ks * p.ldb;
    p.c += (int64_t)blockIdx.y * p.cslice;
    p.K = min(p.kslice, p.K - ks);
  }
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
      if (SPLIT) {
        acc[i][j][0] = 0.0;
        acc[i][j][1] = 0.0;
      } else if (VEC == 2 && row < p.M && col + 1 < p.N) {
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

// ---------------------------------------------------------------------------------------------
// TMA-fed variant.  One elected thread issues the operand tiles with cp.async.bulk.tensor (TMA,
// 64-byte swizzle, out-of-bounds elements zero-filled by the hardware) into a 2-stage ring whose
// "full" mbarriers carry the transaction bytes; the compute warps only wait on the barrier and read
// fragments.  Boxes are 8 doubles (64 B) wide: A stage = BK/8 boxes of [BM][8] (k inner), B stage
// = BN/8 boxes of [BK][8] (n inner).  With the 64-byte swizzle, 16-byte chunk c of box row r lives
// at chunk c ^ ((r >> 1) & 3).  The k slots of each DMMA k-quad are permuted inside every group of
// 8 k values -- thread t of quad q (q = 0, 1) takes k = 2q + (t & 1) + 4 (t >> 1) -- which makes
// every 64-bit fragment load of A and B hit 16 distinct bank pairs per half-warp (the minimum two
// wavefronts per warp).  A and B use the same permutation, so each DMMA sums over 4 distinct k.
struct TmaGemmArgs {
  double* c;
  int64_t ldc, M, N, K;
  int tiles_m, tiles_n;
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  do {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done)
                 : "r"(a), "r"(parity)
                 : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(double* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}

template <class C>
struct TmaCfg {
  static_assert(C::BK % 8 == 0 && C::BN % 8 == 0 && C::TN % 8 == 0, "8-wide boxes");
  static constexpr int ABOX = C::BM * 8, BBOX = C::BK * 8;     // doubles per box
  static constexpr int STAGE = C::BM * C::BK + C::BK * C::BN;  // doubles per stage
  static constexpr int SMEM = C::ST * STAGE * 8 + 64;           // + the stage mbarriers, counters
  static constexpr int MINB = (2 * SMEM <= 227 * 1024) ? 2 : 1;
};

template <class C>
__global__ void __launch_bounds__(C::THREADS, TmaCfg<C>::MINB)
    gemm_dmma_tma(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, TmaGemmArgs p) {
  using T = TmaCfg<C>;
  // no static shared memory: the dynamic block starts at offset 0 (1024-aligned for the swizzle), and
  // fragment loads through `sm` stay LDS (a pointer re-aligned by integer arithmetic would compile
  // to generic loads); the stage barriers sit after the stages
  extern __shared__ __align__(1024) double gt_smem[];
  double* sm = gt_smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(gt_smem + C::ST * T::STAGE);
  int* drained = reinterpret_cast<int*>(full + C::ST);  // per slot: warps done with it
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / C::WN, wn = warp % C::WN;
  int tm, tn;
  tile_coords(blockIdx.x, p.tiles_m, p.tiles_n, tm, tn);
  const int m0 = tm * C::BM, n0 = tn * C::BN;
  const int KT = (int)((p.K + C::BK - 1) / C::BK);
  if (tid == 0) {
    for (int s = 0; s < C::ST; ++s) {
      mbar_init(&full[s], 1);
      drained[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int s, int kt) {  // one thread
    double* st = sm + s * T::STAGE;
    mbar_expect_tx(&full[s], (unsigned)(T::STAGE * 8));
    const int k0 = kt * C::BK;
#pragma unroll
    for (int kb = 0; kb < C::BK / 8; ++kb) tma_load_2d(st + kb * T::ABOX, &ta, k0 + kb * 8, m0, &full[s]);
#pragma unroll
    for (int nb = 0; nb < C::BN / 8; ++nb)
      tma_load_2d(st + C::BM * C::BK + nb * T::BBOX, &tb, n0 + nb * 8, k0, &full[s]);
  };
  if (tid == 0)
    for (int s = 0; s < C::ST && s < KT; ++s) issue(s, s);
  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i) {
    const int64_t row = m0 + wm * C::TM + i * 8 + g;
#pragma unroll
    for (int j = 0; j < C::FN; ++j) {
      const int64_t col = n0 + wn * C::TN + j * 8 + 2 * t;
      const double* cp = p.c + row * p.ldc + col;
      if (row < p.M && col + 1 < p.N) {
        const double2 v = *reinterpret_cast<const double2*>(cp);
        acc[i][j][0] = v.x;
        acc[i][j][1] = v.y;
      } else {
        acc[i][j][0] = (row < p.M && col < p.N) ? cp[0] : 0.0;
        acc[i][j][1] = (row < p.M && col + 1 < p.N) ? cp[1] : 0.0;
      }
    }
  }
  // per-thread fragment offsets (doubles).  k slot of thread t in quad q of an 8-group:
  // kl = 2q + (t & 1) + 4 (t >> 1).  A (box = 8-k group): row m = wm TM + 8i + g, chunk (kl >> 1) ^
  // ((m >> 1) & 3) = (q + 2 (t >> 1)) ^ (g >> 1).  B (box = 8 columns n = wn TN + 8j + g): row kl,
  // chunk (g >> 1) ^ ((kl >> 1) & 3).
  const int tlo = t & 1, thi = t >> 1;
  const int a_base = (wm * C::TM + g) * 8 + tlo;
  const int b_base = (wn * C::TN / 8) * T::BBOX + (g & 1);
  int xa[2], xb[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int h2 = q + 2 * thi;  // kl >> 1
    xa[q] = ((h2 ^ (g >> 1)) << 1);
    xb[q] = (2 * q + tlo + 4 * thi) * 8 + (((g >> 1) ^ h2) << 1);
  }
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % C::ST;
    mbar_wait(&full[s], (unsigned)((kt / C::ST) & 1));
    const double* cA = sm + s * T::STAGE + a_base;
    const double* cB = sm + s * T::STAGE + C::BM * C::BK + b_base;
#pragma unroll
    for (int kb = 0; kb < C::BK / 8; ++kb) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        double af[C::FM], bf[C::FN];
#pragma unroll
        for (int i = 0; i < C::FM; ++i) af[i] = cA[kb * T::ABOX + i * 64 + xa[q]];
#pragma unroll
        for (int j = 0; j < C::FN; ++j) bf[j] = -cB[j * T::BBOX + kb * 64 + xb[q]];
#pragma unroll
        for (int i = 0; i < C::FM; ++i)
#pragma unroll
          for (int j = 0; j < C::FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
    // the last warp to finish slot s refills it (no CTA-wide barrier in the main loop)
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&drained[s], 1) == C::THREADS / 32 - 1) {
        drained[s] = 0;
        if (kt + C::ST < KT) issue(s, kt + C::ST);
      }
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
      if (col + 1 < p.N) {
        *reinterpret_cast<double2*>(cp) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else if (col < p.N) {
        cp[0] = acc[i][j][0];
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Warp-specialised TMA GEMM (the production trailing update).  Per CTA: warpgroup 0 = the producer
// (setmaxnreg.dec; one elected thread streams the A / B stages with cp.async.bulk.tensor into an
// ST-deep ring of full / empty mbarriers), warpgroup 1 = four DMMA consumer warps of 64 x 32
// (setmaxnreg.inc) that only wait on "full", read fragments and release the slot on "empty".  Two
// CTAs per SM: one CTA's C prologue / epilogue overlaps the other's main loop, and the block
// scheduler can hand SMs to the concurrent panel kernel as tiles retire (the look-ahead's
// malleability).  Operand layout and the conflict-free k permutation are those of gemm_dmma_tma.
template <int BM_, int BN_, int BK_, int ST_>
struct WsCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, ST = ST_;
  static constexpr int WM = 2, WN = 2, TM = BM / WM, TN = BN / WN, FM = TM / 8, FN = TN / 8;
  static constexpr int CONSUMERS = WM * WN * 32;
  static constexpr int THREADS = CONSUMERS + 128;  // + the producer warpgroup
  static constexpr int ABOX = BM * 8, BBOX = BK * 8;
  static constexpr int STAGE = BM * BK + BK * BN;            // doubles
  static constexpr int SMEM = ST * STAGE * 8 + 2 * ST * 8;   // + full / empty barriers
  static constexpr int PRODUCER_REGS = 24, CONSUMER_REGS = 232;  // 128 x (24 + 232) = 2 CTAs/SM x 32K
  static_assert(BK % 8 == 0 && BN % 8 == 0 && TN % 8 == 0 && TM % 8 == 0, "8-wide boxes");
  static_assert(2 * SMEM <= 227 * 1024, "two CTAs per SM");
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, 2)
    gemm_dmma_ws(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, TmaGemmArgs p) {
  extern __shared__ __align__(1024) double ws_smem[];
  double* sm = ws_smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(ws_smem + C::ST * C::STAGE);
  uint64_t* empty = full + C::ST;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int tm, tn;
  tile_coords(blockIdx.x, p.tiles_m, p.tiles_n, tm, tn);
  const int m0 = tm * C::BM, n0 = tn * C::BN;
  const int KT = (int)((p.K + C::BK - 1) / C::BK);
  if (tid == 0) {
    for (int s = 0; s < C::ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::CONSUMERS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp < 4) {
    // ---- producer warpgroup: one thread issues every stage, the others retire
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::PRODUCER_REGS));
    if (warp == 0 && lane == 0) {
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % C::ST;
        if (kt >= C::ST) mbar_wait(&empty[s], (unsigned)((kt / C::ST - 1) & 1));
        double* st = sm + s * C::STAGE;
        mbar_expect_tx(&full[s], (unsigned)(C::STAGE * 8));
        const int k0 = kt * C::BK;
#pragma unroll
        for (int kb = 0; kb < C::BK / 8; ++kb) tma_load_2d(st + kb * C::ABOX, &ta, k0 + kb * 8, m0, &full[s]);
#pragma unroll
        for (int nb = 0; nb < C::BN / 8; ++nb)
          tma_load_2d(st + C::BM * C::BK + nb * C::BBOX, &tb, n0 + nb * 8, k0, &full[s]);
      }
    }
    return;
  }
  // ---- consumer warpgroup
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::CONSUMER_REGS));
  const int cw = warp - 4;
  const int g = lane >> 2, t = lane & 3;
  const int wm = cw / C::WN, wn = cw % C::WN;
  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i) {
    const int64_t row = m0 + wm * C::TM + i * 8 + g;
#pragma unroll
    for (int j = 0; j < C::FN; ++j) {
      const int64_t col = n0 + wn * C::TN + j * 8 + 2 * t;
      const double* cp = p.c + row * p.ldc + col;
      if (row < p.M && col + 1 < p.N) {
        const double2 v = *reinterpret_cast<const double2*>(cp);
        acc[i][j][0] = v.x;
        acc[i][j][1] = v.y;
      } else {
        acc[i][j][0] = (row < p.M && col < p.N) ? cp[0] : 0.0;
        acc[i][j][1] = (row < p.M && col + 1 < p.N) ? cp[1] : 0.0;
      }
    }
  }
  // fragment offsets: see gemm_dmma_tma (k slot of thread t in quad q of an 8-group:
  // kl = 2q + (t & 1) + 4 (t >> 1); 64-byte swizzle chunk = (kl >> 1) ^ ((row >> 1) & 3))
  const int tlo = t & 1, thi = t >> 1;
  const int a_base = (wm * C::TM + g) * 8 + tlo;
  const int b_base = (wn * C::TN / 8) * C::BBOX + (g & 1);
  int xa[2], xb[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int h2 = q + 2 * thi;
    xa[q] = ((h2 ^ (g >> 1)) << 1);
    xb[q] = (2 * q + tlo + 4 * thi) * 8 + (((g >> 1) ^ h2) << 1);
  }
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % C::ST;
    mbar_wait(&full[s], (unsigned)((kt / C::ST) & 1));
    const double* cA = sm + s * C::STAGE + a_base;
    const double* cB = sm + s * C::STAGE + C::BM * C::BK + b_base;
#pragma unroll
    for (int kb = 0; kb < C::BK / 8; ++kb) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        double af[C::FM], bf[C::FN];
#pragma unroll
        for (int i = 0; i < C::FM; ++i) af[i] = cA[kb * C::ABOX + i * 64 + xa[q]];
#pragma unroll
        for (int j = 0; j < C::FN; ++j) bf[j] = -cB[j * C::BBOX + kb * 64 + xb[q]];
#pragma unroll
        for (int i = 0; i < C::FM; ++i)
#pragma unroll
          for (int j = 0; j < C::FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
    // release the slot to the producer's next TMA write: the fragment reads above are generic-proxy
    // loads that the compiler issues ahead of their DMMAs (and of this arrive), the refill is an
    // async-proxy write -- order them across proxies first (without the fence, the refill overwrote
    // slots still being read: random wrong 8-row groups with 4+ stages)
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
#pragma unroll
  for (int i = 0; i < C::FM; ++i) {
    const int64_t row = m0 + wm * C::TM + i * 8 + g;
    if (row >= p.M) continue;
#pragma unroll
    for (int j = 0; j < C::FN; ++j) {
      const int64_t col = n0 + wn * C::TN + j * 8 + 2 * t;
      double* cp = p.c + row * p.ldc + col;
      if (col + 1 < p.N) {
        *reinterpret_cast<double2*>(cp) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else if (col < p.N) {
        cp[0] = acc[i][j][0];
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// The same warp-specialised GEMM as a PERSISTENT kernel over an atomic tile queue, for the
// SM-partitioned look-ahead (pflu_options.malleable, the reference's LA / LA_MB):
//   * main grid (ctl.joiner = 0): two CTAs per SM; a CTA on an SM flagged in ctl.mask (the SMs the
//     panel kernel occupies) exits at once, so the panel chain keeps those SMs;
//   * join grid (ctl.joiner = 1, launched on the panel stream after PF(k+1)): the panel's SMs take
//     the remaining tiles of the same queue -- the reference's panel worker rejoining the GEMM team
//     at the next tile boundary (runtime.py:99-113, factor.py:503-504).
// The producer thread pops a tile, streams its K stages through the ring and publishes the tile
// index with the first stage; an exhausted queue is signalled by a data-less arrive on "full".
struct WsCtl {
  int* counter;          // tile queue head (zeroed before the main launch)
  const unsigned* mask;  // reserved-SM bitmask (NULL: none)
  int joiner;
};

template <class C>
__global__ void __launch_bounds__(C::THREADS, 2)
    gemm_dmma_ws_pers(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, TmaGemmArgs p,
                      WsCtl ctl) {
  extern __shared__ __align__(1024) double ws_smem[];
  double* sm = ws_smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(ws_smem + C::ST * C::STAGE);
  uint64_t* empty = full + C::ST;
  int* tile_of = reinterpret_cast<int*>(empty + C::ST);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (!ctl.joiner && ctl.mask) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;\n" : "=r"(smid));
    if ((ctl.mask[smid >> 5] >> (smid & 31)) & 1u) return;  // this SM belongs to the panel chain
  }
  const int ntiles = p.tiles_m * p.tiles_n;
  const int KT = (int)((p.K + C::BK - 1) / C::BK);
  if (tid == 0) {
    for (int s = 0; s < C::ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::CONSUMERS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::PRODUCER_REGS));
    if (warp == 0 && lane == 0) {
      int g = 0;
      for (;;) {
        const int tile = atomicAdd(ctl.counter, 1);
        const bool done = tile >= ntiles;
        int tm = 0, tn = 0;
        if (!done) tile_coords(tile, p.tiles_m, p.tiles_n, tm, tn);
        for (int kt = 0; kt < (done ? 1 : KT); ++kt, ++g) {
          const int s = g % C::ST;
          if (g >= C::ST) mbar_wait(&empty[s], (unsigned)((g / C::ST - 1) & 1));
          if (kt == 0) tile_of[s] = done ? -1 : tile;
          if (done) {
            mbar_arrive(&full[s]);
            break;
          }
          double* st = sm + s * C::STAGE;
          mbar_expect_tx(&full[s], (unsigned)(C::STAGE * 8));
          const int k0 = kt * C::BK;
#pragma unroll
          for (int kb = 0; kb < C::BK / 8; ++kb) tma_load_2d(st + kb * C::ABOX, &ta, k0 + kb * 8, tm * C::BM, &full[s]);
#pragma unroll
          for (int nb = 0; nb < C::BN / 8; ++nb)
            tma_load_2d(st + C::BM * C::BK + nb * C::BBOX, &tb, tn * C::BN + nb * 8, k0, &full[s]);
        }
        if (done) break;
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::CONSUMER_REGS));
  const int cw = warp - 4;
  const int g8 = lane >> 2, t = lane & 3;
  const int wm = cw / C::WN, wn = cw % C::WN;
  const int tlo = t & 1, thi = t >> 1;
  const int a_base = (wm * C::TM + g8) * 8 + tlo;
  const int b_base = (wn * C::TN / 8) * C::BBOX + (g8 & 1);
  int xa[2], xb[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int h2 = q + 2 * thi;
    xa[q] = ((h2 ^ (g8 >> 1)) << 1);
    xb[q] = (2 * q + tlo + 4 * thi) * 8 + (((g8 >> 1) ^ h2) << 1);
  }
  int g = 0;
  for (;;) {
    mbar_wait(&full[g % C::ST], (unsigned)((g / C::ST) & 1));
    const int tile = tile_of[g % C::ST];
    if (tile < 0) break;
    int tm, tn;
    tile_coords(tile, p.tiles_m, p.tiles_n, tm, tn);
    const int m0 = tm * C::BM, n0 = tn * C::BN;
    double acc[C::FM][C::FN][2];
#pragma unroll
    for (int i = 0; i < C::FM; ++i) {
      const int64_t row = m0 + wm * C::TM + i * 8 + g8;
#pragma unroll
      for (int j = 0; j < C::FN; ++j) {
        const int64_t col = n0 + wn * C::TN + j * 8 + 2 * t;
        const double* cp = p.c + row * p.ldc + col;
        if (row < p.M && col + 1 < p.N) {
          const double2 v = *reinterpret_cast<const double2*>(cp);
          acc[i][j][0] = v.x;
          acc[i][j][1] = v.y;
        } else {
          acc[i][j][0] = (row < p.M && col < p.N) ? cp[0] : 0.0;
          acc[i][j][1] = (row < p.M && col + 1 < p.N) ? cp[1] : 0.0;
        }
      }
    }
    for (int kt = 0; kt < KT; ++kt, ++g) {
      const int s = g % C::ST;
      if (kt > 0) mbar_wait(&full[s], (unsigned)((g / C::ST) & 1));
      const double* cA = sm + s * C::STAGE + a_base;
      const double* cB = sm + s * C::STAGE + C::BM * C::BK + b_base;
#pragma unroll
      for (int kb = 0; kb < C::BK / 8; ++kb) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          double af[C::FM], bf[C::FN];
#pragma unroll
          for (int i = 0; i < C::FM; ++i) af[i] = cA[kb * C::ABOX + i * 64 + xa[q]];
#pragma unroll
          for (int j = 0; j < C::FN; ++j) bf[j] = -cB[j * C::BBOX + kb * 64 + xb[q]];
#pragma unroll
          for (int i = 0; i < C::FM; ++i)
#pragma unroll
            for (int j = 0; j < C::FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // see gemm_dmma_ws
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
#pragma unroll
    for (int i = 0; i < C::FM; ++i) {
      const int64_t row = m0 + wm * C::TM + i * 8 + g8;
      if (row >= p.M) continue;
#pragma unroll
      for (int j = 0; j < C::FN; ++j) {
        const int64_t col = n0 + wn * C::TN + j * 8 + 2 * t;
        double* cp = p.c + row * p.ldc + col;
        if (col + 1 < p.N) {
          *reinterpret_cast<double2*>(cp) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else if (col < p.N) {
          cp[0] = acc[i][j][0];
        }
      }
    }
  }
}

// measured at the C4 step-0 shape 32512 x 32512 x 256 (tools/gemm_ws_probe.py, profiles/r05_gemm_ws.log):
// WS1 35.4 TFLOP/s (production), WS2 35.2, WS0 35.0, WS3 34.3; cp.async GV6 33.7.  An L2 prefetch of
// the C tile by the idle producer warps made WS1 / WS0 slower (34.1 / 33.8).
using WS0 = WsCfg<128, 64, 16, 4>;  // 4 stages of K = 16 (24 KB each), 2 CTAs/SM
using WS1 = WsCfg<128, 64, 32, 2>;  // 2 stages of K = 32 (48 KB each) -- production
using WS2 = WsCfg<128, 64, 16, 3>;  // 3 stages of K = 16
using WS3 = WsCfg<128, 64, 8, 8>;   // 8 stages of K = 8

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
using GV9 = GemmCfg<128, 32, 16, 2, 2, 1>;   // 2 warps of 64x32 per CTA, 40 KB: 4 independent CTAs/SM

}  // namespace pflu
