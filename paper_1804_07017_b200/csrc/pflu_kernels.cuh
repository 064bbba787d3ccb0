// pflu_kernels.cuh -- sm_100a device kernels for blocked LU with partial pivoting.
//
// Storage: ROW-MAJOR float64, element (i, j) at a[i * lda + j].  Rows are contiguous, so every
// row interchange is a coalesced (128-bit when aligned) row copy and the trailing update's
// operands are "K-contiguous" L21 rows and "N-contiguous" U12 rows.
//
// Kernels (reference functions they replace, pkg/src/panelforge/...):
//   pivot_plan_kernel   _jit.py:141-151 laswp_run   -- composes b ascending swaps into a gather plan
//   swap_trsm_kernel    _jit.py:141-151 + 104-113   -- laswp (gather/scatter by plan) fused with the
//                       unit-lower triangular solve of the U12 block row
//   trsm_kernel         _jit.py:104-113              -- in-panel unit-lower solve (no swaps)
//   gemm_exact_kernel   _jit.py:54-80 macro_run      -- C -= A*B in the reference rounding (mul, then sub)
// The DMMA trailing-update GEMM lives in pflu_gemm.cuh, the panel kernel in pflu_panel.cuh.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pflu {

// ------------------------------------------------------------------------------------------
// small helpers

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Reference rounding: multiply, round, subtract, round (no FMA contraction).  _jit.py:183-186.
__device__ __forceinline__ double sub_mul_exact(double c, double a, double b) {
  return __dsub_rn(c, __dmul_rn(a, b));
}

// ------------------------------------------------------------------------------------------
// Pivot key: reproduces the sequential scan of _jit.py:163-170 (start with the diagonal, take a
// row only if STRICTLY greater, so ties go to the smallest row and NaNs are never taken unless
// the diagonal itself is NaN, in which case the diagonal is kept).

__device__ __forceinline__ double pivot_key(double x, bool is_diag) {
  double v = fabs(x);
  if (v != v) return is_diag ? __longlong_as_double(0x7ff0000000000000ll) : -1.0;
  return v;
}
// better(a, b): larger key wins; equal keys -> smaller row.
__device__ __forceinline__ bool key_better(double ka, long long ra, double kb, long long rb) {
  return ka > kb || (ka == kb && ra < rb);
}

// Order-preserving map of a (non-NaN) double onto uint64.
__device__ __forceinline__ unsigned long long key_ord(double k) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(k);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
// Warp arg-max under key_better (largest key, equal keys -> smallest row) with redux.sync: every
// lane receives the winner; returns the winning lane (for extra payload).  Rows are >= 0.
__device__ __forceinline__ int warp_best(double& k, long long& r) {
  const unsigned full = 0xffffffffu;
  __syncwarp();  // callers may arrive from lane-divergent code: reconverge before the collectives
  const unsigned long long u = key_ord(k);
  const unsigned hi = (unsigned)(u >> 32), lo = (unsigned)u;
  const unsigned mhi = __reduce_max_sync(full, hi);
  const unsigned mlo = __reduce_max_sync(full, hi == mhi ? lo : 0u);
  const unsigned eq = __ballot_sync(full, hi == mhi && lo == mlo);
  int src = __ffs(eq) - 1;
  if (eq & (eq - 1)) {  // bitwise-equal best keys in several lanes: the smallest row
    const unsigned long long rr = ((eq >> (threadIdx.x & 31)) & 1u) ? (unsigned long long)r : ~0ull;
    const unsigned rhi = (unsigned)(rr >> 32), rlo = (unsigned)rr;
    const unsigned nhi = __reduce_min_sync(full, rhi);
    const unsigned nlo = __reduce_min_sync(full, rhi == nhi ? rlo : ~0u);
    src = __ffs(__ballot_sync(full, rhi == nhi && rlo == nlo)) - 1;
  }
  k = __shfl_sync(full, k, src);
  r = __shfl_sync(full, r, src);
  return src;
}

// Integer pivot keys (the v2 panel exchange): order-preserving for |x|, with "no candidate" < NaN off the
// diagonal < every magnitude; a NaN on the diagonal ranks as +inf (the scan of _jit.py:163-170 keeps it).
constexpr unsigned long long ORD_NONE = 0ull, ORD_NAN = 1ull, ORD_ZERO = 0x8000000000000000ull;
__device__ __forceinline__ unsigned long long pivot_key_ord(double x, bool is_diag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
  if (b > 0x7ff0000000000000ull) return is_diag ? 0xfff0000000000000ull : ORD_NAN;
  return b | ORD_ZERO;
}
// Warp max of a 96-bit (hi, mid, lo) tuple, lexicographic: three redux.sync, the result lands in every
// lane (uniform registers) without shuffles or a tie branch.  The v2 panel exchange packs (integer key,
// ~row) so that the largest tuple is the largest key and, among equal keys, the smallest row.
__device__ __forceinline__ void warp_max96(unsigned& h, unsigned& m, unsigned& l) {
  const unsigned full = 0xffffffffu;
  __syncwarp();
  const unsigned mh = __reduce_max_sync(full, h);
  const bool e1 = h == mh;
  const unsigned mm = __reduce_max_sync(full, e1 ? m : 0u);
  const unsigned ml = __reduce_max_sync(full, (e1 & (m == mm)) ? l : 0u);
  h = mh; m = mm; l = ml;
}
// branch-free lane-local max of two such tuples
__device__ __forceinline__ void max96(unsigned long long& K, unsigned& l, unsigned long long K2, unsigned l2) {
  const bool gt = (K2 > K) | ((K2 == K) & (l2 > l));
  K = gt ? K2 : K;
  l = gt ? l2 : l;
}

// ==========================================================================================
// Pivot plan: composes the ascending LAPACK swaps piv[d..d+np) (global 0-based rows, piv[i] >= i)
// into a gather.  Output layout (int64): [0] = E (extra rows), [1 .. np] = source row of top row
// d+i, then E (dst, src) pairs for rows >= d+np.  Extra rows only ever receive original top-row
// data (a row >= d+np is only swapped with top rows), top rows may receive either.

constexpr int PLAN_MAX = 1024;

// Parallel composition.  With piv[i] >= i (LAPACK getrf), let g(i) be the original row whose data
// sits in row d+i just before swap i.  Row d+i only changes before step i when an earlier swap
// targets it, so g(i) = g(pt(i)) with pt(i) = last i' < i with piv[i'] = d+i, else g(i) = d+i.
// Then (PA)[d+i] = A[src(i)] with src(i) = g(i) if piv[i] == d+i, else g(ps(i)) for
// ps(i) = last i' < i with piv[i'] == piv[i], else the original row piv[i].  An extra row R >= d+np
// finally holds g(last i with piv[i] == R).  pt() chains are resolved by pointer jumping.
// General laswp (pflu_laswp) may pass piv[i] < d+i; then the sequential fallback is used.
__global__ void __launch_bounds__(256) pivot_plan_kernel(const int64_t* __restrict__ piv, int64_t d,
                                                          int np, int64_t* __restrict__ plan) {
  __shared__ long long spiv[PLAN_MAX];
  __shared__ int ptr_[PLAN_MAX];
  __shared__ long long g[PLAN_MAX];
  __shared__ int flags[2];
  const int tid = threadIdx.x;
  const long long top_end = d + np;
  if (tid == 0) { flags[0] = 0; flags[1] = 0; }
  for (int i = tid; i < np; i += blockDim.x) spiv[i] = piv[d + i];
  for (int i = tid; i < np; i += blockDim.x) ptr_[i] = -1;
  __syncthreads();
  for (int i = tid; i < np; i += blockDim.x)
    if (spiv[i] < d + i) flags[1] = 1;  // not a getrf pivot sequence
  __syncthreads();
  if (flags[1] == 0) {
    // pt(i): atomicMax over earlier swaps targeting top row d+i (only i' <= i can target it)
    for (int i = tid; i < np; i += blockDim.x) {
      const long long r = spiv[i];
      if (r < top_end && r != d + i) atomicMax(&ptr_[(int)(r - d)], i);
    }
    __syncthreads();
    for (int i = tid; i < np; i += blockDim.x) g[i] = ptr_[i] < 0 ? d + i : -1;
    __syncthreads();
    // pointer jumping: g[i] = g[ptr[i]] until resolved (chains strictly decrease the index)
    for (int round = 0; round < 12; ++round) {
      if (tid == 0) flags[0] = 0;
      __syncthreads();
      for (int i = tid; i < np; i += blockDim.x) {
        if (g[i] < 0) {
          const int p = ptr_[i];
          if (g[p] >= 0) g[i] = g[p];
          else { ptr_[i] = ptr_[p]; flags[0] = 1; }
        }
      }
      __syncthreads();
      if (flags[0] == 0) break;
      __syncthreads();
    }
    __shared__ int s_ne;
    if (tid == 0) s_ne = 0;
    __syncthreads();
    for (int i = tid; i < np; i += blockDim.x) {
      const long long r = spiv[i];
      int ps = -1, nxt = -1;
      for (int k = 0; k < np; ++k) {
        if (spiv[k] == r) {
          if (k < i) ps = k;
          else if (k > i && nxt < 0) nxt = k;
        }
      }
      long long src;
      if (r == d + i) src = g[i];
      else if (ps >= 0) src = g[ps];
      else src = r;
      plan[1 + i] = src;
      if (r >= top_end && nxt < 0) {  // last swap into extra row r
        const int e = atomicAdd(&s_ne, 1);
        plan[1 + np + 2 * e] = r;
        plan[1 + np + 2 * e + 1] = g[i];
      }
    }
    __syncthreads();
    if (tid == 0) plan[0] = s_ne;
    return;
  }
  // sequential fallback (general laswp pivots): slots for rows outside [d, d+np)
  __shared__ int first_occ[PLAN_MAX];
  __shared__ int ext_first[PLAN_MAX];
  __shared__ int slot_of[PLAN_MAX];
  __shared__ int contents[2 * PLAN_MAX];
  __shared__ int s_ne2;
  for (int i = tid; i < np; i += blockDim.x) {
    const long long r = spiv[i];
    int fo = -1;
    if (r < d || r >= top_end) {
      fo = i;
      for (int k = 0; k < i; ++k)
        if (spiv[k] == r) { fo = k; break; }
    }
    first_occ[i] = fo;
  }
  __syncthreads();
  if (tid == 0) {
    int ne = 0;
    for (int i = 0; i < np; ++i)
      if (first_occ[i] == i) { ext_first[ne] = i; ptr_[i] = np + ne; ++ne; }
    s_ne2 = ne;
  }
  __syncthreads();
  const int ne = s_ne2;
  for (int i = tid; i < np; i += blockDim.x) {
    const long long r = spiv[i];
    slot_of[i] = (r >= d && r < top_end) ? (int)(r - d) : ptr_[first_occ[i]];
  }
  for (int s2 = tid; s2 < np + ne; s2 += blockDim.x) contents[s2] = s2;
  __syncthreads();
  if (tid == 0) {
    for (int i = 0; i < np; ++i) {
      const int s2 = slot_of[i];
      if (s2 != i) { const int t = contents[i]; contents[i] = contents[s2]; contents[s2] = t; }
    }
  }
  __syncthreads();
  auto row_of = [&](int s2) -> long long { return s2 < np ? d + s2 : spiv[ext_first[s2 - np]]; };
  if (tid == 0) plan[0] = ne;
  for (int i = tid; i < np; i += blockDim.x) plan[1 + i] = row_of(contents[i]);
  for (int e = tid; e < ne; e += blockDim.x) {
    plan[1 + np + 2 * e] = row_of(np + e);
    plan[1 + np + 2 * e + 1] = row_of(contents[np + e]);
  }
}

// ==========================================================================================
// Unit-lower triangular solve of a TW-column tile held in shared memory:
//   X (np x TW, row-major in smem) := unit_lower(L)^-1 X,  L global (leading dimension ldl).
// Exact reference order (_jit.py:109-113): every x_r takes x_r -= L_ri * x_i for i ascending,
// multiply then subtract.  Blocked by DB = TW rows: the DB x DB diagonal block is solved in
// registers by TW threads (one column each, no barriers), then the rows below are updated from an
// smem-staged L panel with 4 independent rows per thread in flight.  Lst: >= max(np, TW) * TW doubles.

template <int TW>
__device__ __forceinline__ void tile_trsm_smem(double* X, double* Lst, const double* __restrict__ L, int64_t ldl,
                                               int np) {
  constexpr int DB = TW;
  constexpr int RL = 256 / TW;
  const int tid = threadIdx.x, col = tid % TW, rl = tid / TW;
  for (int ib = 0; ib < np; ib += DB) {
    const int nb = min(DB, np - ib);
    const int nrows = np - ib;
    __syncthreads();  // previous readers of Lst / writers of X are done
    for (int idx = tid; idx < nrows * DB; idx += 256) {
      const int r = idx / DB, i = idx - r * DB;
      Lst[idx] = (i < nb) ? L[(int64_t)(ib + r) * ldl + ib + i] : 0.0;
    }
    __syncthreads();
    if (tid < TW) {
      double x[DB];
#pragma unroll
      for (int i = 0; i < DB; ++i) x[i] = (i < nb) ? X[(ib + i) * TW + col] : 0.0;
#pragma unroll
      for (int i = 0; i < DB; ++i) {
#pragma unroll
        for (int r = i + 1; r < DB; ++r) x[r] = sub_mul_exact(x[r], Lst[r * DB + i], x[i]);
      }
#pragma unroll
      for (int i = 0; i < DB; ++i)
        if (i < nb) X[(ib + i) * TW + col] = x[i];
    }
    __syncthreads();
    if (ib + nb < np) {
      double xi[DB];
#pragma unroll
      for (int i = 0; i < DB; ++i) xi[i] = (i < nb) ? X[(ib + i) * TW + col] : 0.0;
      int r = ib + nb + rl;
      for (; r + 3 * RL < np; r += 4 * RL) {
        double y0 = X[r * TW + col], y1 = X[(r + RL) * TW + col];
        double y2 = X[(r + 2 * RL) * TW + col], y3 = X[(r + 3 * RL) * TW + col];
        const double* l0 = Lst + (r - ib) * DB;
#pragma unroll
        for (int i = 0; i < DB; ++i) {
          y0 = sub_mul_exact(y0, l0[i], xi[i]);
          y1 = sub_mul_exact(y1, l0[RL * DB + i], xi[i]);
          y2 = sub_mul_exact(y2, l0[2 * RL * DB + i], xi[i]);
          y3 = sub_mul_exact(y3, l0[3 * RL * DB + i], xi[i]);
        }
        X[r * TW + col] = y0;
        X[(r + RL) * TW + col] = y1;
        X[(r + 2 * RL) * TW + col] = y2;
        X[(r + 3 * RL) * TW + col] = y3;
      }
      for (; r < np; r += RL) {
        double y0 = X[r * TW + col];
        const double* l0 = Lst + (r - ib) * DB;
#pragma unroll
        for (int i = 0; i < DB; ++i) y0 = sub_mul_exact(y0, l0[i], xi[i]);
        X[r * TW + col] = y0;
      }
    }
  }
  __syncthreads();
}

// K2/K3: laswp by plan, optionally fused with the unit-lower triangular solve of the top block
// (U12 := L11^-1 * P * A12).  One CTA per TW-column tile of [c0, c1).  All reads of original
// values complete (barrier) before any write, so the in-place permutation is race free.
// Smem: X [np][TW] (new top block) + E [max(np, 1024/TW)][TW] (extra rows, then the L panel).

template <int TW>
__global__ void __launch_bounds__(256) swap_trsm_kernel(double* __restrict__ a, int64_t lda, int64_t d,
                                                         int np, const int64_t* __restrict__ plan,
                                                         int64_t c0, int64_t c1,
                                                         const double* __restrict__ L, int64_t ldl,
                                                         int do_trsm) {
  extern __shared__ double st_smem[];
  constexpr int RL = 256 / TW;
  const int tid = threadIdx.x;
  const int col = tid % TW;
  const int rl = tid / TW;
  const int64_t cb = c0 + (int64_t)blockIdx.x * TW;
  const int64_t gc = cb + col;
  const bool cok = gc < c1;
  const int ne = (int)plan[0];
  double* X = st_smem;              // [np][TW] new top block
  double* E = st_smem + np * TW;    // [ne][TW] values for extra rows, later the staged L panel
  // gathers in batches of 8 independent (plan, row) loads per thread
  constexpr int GB = 8;
  for (int i0 = rl; i0 < np; i0 += GB * RL) {
    int64_t src[GB];
    double v[GB];
#pragma unroll
    for (int u = 0; u < GB; ++u) src[u] = i0 + u * RL < np ? plan[1 + i0 + u * RL] : 0;
#pragma unroll
    for (int u = 0; u < GB; ++u) v[u] = (cok && i0 + u * RL < np) ? a[src[u] * lda + gc] : 0.0;
#pragma unroll
    for (int u = 0; u < GB; ++u)
      if (i0 + u * RL < np) X[(i0 + u * RL) * TW + col] = v[u];
  }
  for (int e0 = rl; e0 < ne; e0 += GB * RL) {
    int64_t src[GB];
    double v[GB];
#pragma unroll
    for (int u = 0; u < GB; ++u) src[u] = e0 + u * RL < ne ? plan[1 + np + 2 * (e0 + u * RL) + 1] : 0;
#pragma unroll
    for (int u = 0; u < GB; ++u) v[u] = (cok && e0 + u * RL < ne) ? a[src[u] * lda + gc] : 0.0;
#pragma unroll
    for (int u = 0; u < GB; ++u)
      if (e0 + u * RL < ne) E[(e0 + u * RL) * TW + col] = v[u];
  }
  __syncthreads();
  if (cok)
    for (int e = rl; e < ne; e += RL) a[plan[1 + np + 2 * e] * lda + gc] = E[e * TW + col];
  if (do_trsm) tile_trsm_smem<TW>(X, E, L, ldl, np);
  else __syncthreads();
  if (cok)
    for (int i = rl; i < np; i += RL) a[(d + i) * lda + gc] = X[i * TW + col];
}

// Plain unit-lower solve X := unit_lower(L)^-1 X (no swaps), X = np rows x [0, ncols) columns.
template <int TW>
__global__ void __launch_bounds__(256) trsm_kernel(const double* __restrict__ L, int64_t ldl,
                                                    double* __restrict__ Xg, int64_t ldx, int np,
                                                    int64_t ncols) {
  extern __shared__ double st_smem[];
  constexpr int RL = 256 / TW;
  const int tid = threadIdx.x;
  const int col = tid % TW;
  const int rl = tid / TW;
  const int64_t gc = (int64_t)blockIdx.x * TW + col;
  const bool cok = gc < ncols;
  double* X = st_smem;
  double* Lst = st_smem + np * TW;
  for (int i = rl; i < np; i += RL) X[i * TW + col] = cok ? Xg[i * ldx + gc] : 0.0;
  tile_trsm_smem<TW>(X, Lst, L, ldl, np);
  if (cok)
    for (int i = rl; i < np; i += RL) Xg[i * ldx + gc] = X[i * TW + col];
}

// ==========================================================================================
// K4: trailing update C(MxN) -= A(MxK) * B(KxN), all row-major views into the matrix.
// CTA tile 128x64, 4 warps (2x2), warp tile 64x32 = 8x4 DMMA 8x8x4 blocks, K staged 16 at a
// time through a 4-deep cp.async pipeline with XOR-swizzled shared tiles (conflict-free 64-bit
// fragment loads).  Accumulators are seeded from C (like macro_run, _jit.py:70-72); the B
// fragment is negated (exact) so the tensor core computes c + a*(-b) == c - a*b.

constexpr int GM_BM = 128, GM_BN = 64, GM_BK = 16, GM_ST = 4, GM_THREADS = 128;
constexpr int GM_GROUP = 8;
constexpr int GM_SMEM = GM_ST * (GM_BM * GM_BK + GM_BK * GM_BN) * 8;

struct GemmArgs {
  double* c;
  const double* a;
  const double* b;
  int64_t ldc, lda, ldb, M, N, K;
  int tiles_m, tiles_n;
  int64_t kslice, cslice;  // split-K GEMM (QR): K per blockIdx.y slice, C elements between slices
};

__device__ __forceinline__ void tile_coords(int lin, int tiles_m, int tiles_n, int& tm, int& tn) {
  const int per_group = GM_GROUP * tiles_n;
  const int gid = lin / per_group;
  const int first_m = gid * GM_GROUP;
  const int gsize = min(tiles_m - first_m, GM_GROUP);
  const int r = lin - gid * per_group;
  tm = first_m + r % gsize;
  tn = r / gsize;
}

template <int VEC>
__device__ __forceinline__ void gemm_load_stage(const GemmArgs& p, double* sA, double* sB, int m0, int n0,
                                                int64_t k0, int tid) {
  if constexpr (VEC == 2) {
#pragma unroll
    for (int i = 0; i < (GM_BM * GM_BK / 2) / GM_THREADS; ++i) {
      int q = tid + i * GM_THREADS;
      int row = q >> 3, k = (q & 7) * 2;
      int64_t gm = m0 + row, gk = k0 + k;
      int bytes = gm < p.M ? (int)max((int64_t)0, min((int64_t)16, (p.K - gk) * 8)) : 0;
      const double* src = bytes ? p.a + gm * p.lda + gk : p.a;
      cp_async16(sA + row * GM_BK + (k ^ ((row & 3) << 2)), src, bytes);
    }
#pragma unroll
    for (int i = 0; i < (GM_BK * GM_BN / 2) / GM_THREADS; ++i) {
      int q = tid + i * GM_THREADS;
      int kr = q >> 5, n = (q & 31) * 2;
      int64_t gk = k0 + kr, gn = n0 + n;
      int bytes = gk < p.K ? (int)max((int64_t)0, min((int64_t)16, (p.N - gn) * 8)) : 0;
      const double* src = bytes ? p.b + gk * p.ldb + gn : p.b;
      cp_async16(sB + kr * GM_BN + (n ^ ((kr & 3) << 2)), src, bytes);
    }
  } else {
#pragma unroll
    for (int i = 0; i < (GM_BM * GM_BK) / GM_THREADS; ++i) {
      int q = tid + i * GM_THREADS;
      int row = q >> 4, k = q & 15;
      int64_t gm = m0 + row, gk = k0 + k;
      int bytes = (gm < p.M && gk < p.K) ? 8 : 0;
      const double* src = bytes ? p.a + gm * p.lda + gk : p.a;
      cp_async8(sA + row * GM_BK + (k ^ ((row & 3) << 2)), src, bytes);
    }
#pragma unroll
    for (int i = 0; i < (GM_BK * GM_BN) / GM_THREADS; ++i) {
      int q = tid + i * GM_THREADS;
      int kr = q >> 6, n = q & 63;
      int64_t gk = k0 + kr, gn = n0 + n;
      int bytes = (gk < p.K && gn < p.N) ? 8 : 0;
      const double* src = bytes ? p.b + gk * p.ldb + gn : p.b;
      cp_async8(sB + kr * GM_BN + (n ^ ((kr & 3) << 2)), src, bytes);
    }
  }
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Same tiling and pipeline, SIMT arithmetic in the reference's rounding: per element p ascending,
// c = c - a*b with the product rounded first (_jit.py:73-77).  Bitwise equal to the reference.
template <int VEC>
__global__ void __launch_bounds__(GM_THREADS, 2) gemm_exact_kernel(GemmArgs p) {
  extern __shared__ __align__(128) double gm_smem[];
  double* sA = gm_smem;
  double* sB = gm_smem + GM_ST * GM_BM * GM_BK;
  const int tid = threadIdx.x;
  const int tr = tid >> 3;  // 16 row groups of 8 rows (strided by 16)
  const int tc = tid & 7;   // 8 col groups of 8 cols (strided by 8)
  int tm, tn;
  tile_coords(blockIdx.x, p.tiles_m, p.tiles_n, tm, tn);
  const int m0 = tm * GM_BM, n0 = tn * GM_BN;
  const int KT = (int)((p.K + GM_BK - 1) / GM_BK);
#pragma unroll
  for (int s = 0; s < GM_ST - 1; ++s) {
    if (s < KT) gemm_load_stage<VEC>(p, sA + s * GM_BM * GM_BK, sB + s * GM_BK * GM_BN, m0, n0, (int64_t)s * GM_BK, tid);
    cp_async_commit();
  }
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = m0 + tr + 16 * i;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t col = n0 + tc + 8 * j;
      acc[i][j] = (row < p.M && col < p.N) ? p.c[row * p.ldc + col] : 0.0;
    }
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<GM_ST - 2>();
    __syncthreads();
    {
      const int nk = kt + GM_ST - 1;
      const int s = nk % GM_ST;
      if (nk < KT) gemm_load_stage<VEC>(p, sA + s * GM_BM * GM_BK, sB + s * GM_BK * GM_BN, m0, n0, (int64_t)nk * GM_BK, tid);
      cp_async_commit();
    }
    const double* cA = sA + (kt % GM_ST) * GM_BM * GM_BK;
    const double* cB = sB + (kt % GM_ST) * GM_BK * GM_BN;
    const int kmax = (int)min((int64_t)GM_BK, p.K - (int64_t)kt * GM_BK);
    for (int k = 0; k < kmax; ++k) {
      double av[8], bv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = tr + 16 * i;
        av[i] = cA[row * GM_BK + (k ^ ((row & 3) << 2))];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int col = tc + 8 * j;
        bv[j] = cB[k * GM_BN + (col ^ ((k & 3) << 2))];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = sub_mul_exact(acc[i][j], av[i], bv[j]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = m0 + tr + 16 * i;
    if (row >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t col = n0 + tc + 8 * j;
      if (col < p.N) p.c[row * p.ldc + col] = acc[i][j];
    }
  }
}

// ------------------------------------------------------------------------------------------
// Fast-mode (DMMA) laswp + unit-lower solve of the U12 block row, for np <= 256.
//
// diag_inv_kernel: the 32x32 diagonal blocks of L11 inverted once per step (one warp per block, lane j:
// column j by forward substitution).  inv[blk][32][32], row-major, identity-padded past np.
// swap_trsm_dmma_kernel: one CTA per 32-column strip; X = P * A12 strip (256 x 32) in shared
// memory, then per 32-row block i:  X_i := inv(L_ii) X_i,  X_{>i} -= L_{>i,i} X_i  -- both on the
// tensor cores (DMMA 8x8x4), L streamed from L2.  Not bitwise: exact mode keeps swap_trsm_kernel.

// NPMAX rows x BN-column strip, rows padded to BN + 4 doubles (conflict-free B fragments; 32-wide
// strips also conflict-free A/C).  (256, 32): 74 KB, 3 CTAs/SM; (512, 16): 82 KB, 2 CTAs/SM.
template <int NPMAX, int BN>
struct SdCfg {
  static constexpr int LDX = BN + 4;
  static constexpr int SMEM = NPMAX * LDX * 8;
  static constexpr int MINB = (227 * 1024) / (SMEM + 1024) >= 3 ? 3 : 2;
};

__global__ void __launch_bounds__(128) diag_inv_kernel(const double* __restrict__ L, int64_t ldl, int np,
                                                       double* __restrict__ inv) {
  __shared__ double lb[4][32][33];  // grid (2), 4 warps per CTA: one 32x32 block per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int blk = blockIdx.x * 4 + warp; blk * 32 < np; blk += 4 * gridDim.x) {
    const int r0 = blk * 32, nb = min(32, np - r0);
    for (int i = 0; i < 32; ++i)
      lb[warp][i][lane] = (i < nb && lane < nb) ? L[(int64_t)(r0 + i) * ldl + r0 + lane] : 0.0;
    __syncwarp();
    // column `lane` of inv(unit lower): x_i = delta_ij - sum_{k<i} L_ik x_k
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      double s = (i == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k) s = fma(-lb[warp][i][k], x[k], s);
      x[i] = s;
    }
    double* out = inv + (size_t)blk * 1024;
#pragma unroll
    for (int i = 0; i < 32; ++i) out[i * 32 + lane] = x[i];
    __syncwarp();
  }
}

template <int NPMAX, int SD_BN>
__global__ void __launch_bounds__(256, (SdCfg<NPMAX, SD_BN>::MINB)) swap_trsm_dmma_kernel(double* __restrict__ a, int64_t lda, int64_t d,
                                                              int np, const int64_t* __restrict__ plan,
                                                              int64_t c0, int64_t c1,
                                                              const double* __restrict__ L, int64_t ldl,
                                                              const double* __restrict__ inv) {
  extern __shared__ double sd_smem[];
  constexpr int SD_LDX = SdCfg<NPMAX, SD_BN>::LDX;
  constexpr int NBK = SD_BN / 8;  // 8-column DMMA blocks per strip
  double* X = sd_smem;  // [NPMAX][SD_LDX]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int col = tid % SD_BN, rl = tid / SD_BN;  // loads: 8 rows per pass
  constexpr int RL = 256 / SD_BN;
  const int64_t gc = c0 + (int64_t)blockIdx.x * SD_BN + col;
  const bool cok = gc < c1;
  const int ne = (int)plan[0];
  // ---- laswp by plan: gather the new top block, extra rows staged in registers; fully unrolled
  // so that all plan and row loads of a thread are in flight together
  constexpr int EMAX = NPMAX / RL;
  {
    int64_t src[EMAX];
#pragma unroll
    for (int it = 0; it < EMAX; ++it) {
      const int i = rl + it * RL;
      src[it] = i < np ? plan[1 + i] : 0;
    }
    double xv[EMAX];
#pragma unroll
    for (int it = 0; it < EMAX; ++it) {
      const int i = rl + it * RL;
      xv[it] = (cok && i < np) ? a[src[it] * lda + gc] : 0.0;
    }
#pragma unroll
    for (int it = 0; it < EMAX; ++it) X[(rl + it * RL) * SD_LDX + col] = xv[it];
  }
  double ev[EMAX];
  {
    int64_t src[EMAX];
#pragma unroll
    for (int it = 0; it < EMAX; ++it) {
      const int e = rl + it * RL;
      src[it] = e < ne ? plan[1 + np + 2 * e + 1] : 0;
    }
#pragma unroll
    for (int it = 0; it < EMAX; ++it) {
      const int e = rl + it * RL;
      ev[it] = (cok && e < ne) ? a[src[it] * lda + gc] : 0.0;
    }
  }
  __syncthreads();  // every original value read before any row is overwritten
  if (cok) {
#pragma unroll
    for (int it = 0; it < EMAX; ++it) {
      const int e = rl + it * RL;
      if (e < ne) a[plan[1 + np + 2 * e] * lda + gc] = ev[it];
    }
  }
  // ---- blocked solve on DMMA
  const int g = lane >> 2, t = lane & 3;
  const int nblk = (np + 31) / 32;
  for (int ib = 0; ib < nblk; ++ib) {
    const int rb = ib * 32;
    {  // X_i := inv(L_ii) X_i: 4 x NBK 8x8 output blocks, NBK / 2 per warp
      constexpr int JB = NBK / 2;
      const int gg = warp >> 1, nb0 = (warp & 1) * JB;
      const double* iv = inv + (size_t)ib * 1024 + (gg * 8 + g) * 32;
      double acc[JB][2];
#pragma unroll
      for (int j = 0; j < JB; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
      for (int k4 = 0; k4 < 32; k4 += 4) {
        const double av = iv[k4 + t];
#pragma unroll
        for (int j = 0; j < JB; ++j) dmma884(acc[j][0], acc[j][1], av, X[(rb + k4 + t) * SD_LDX + (nb0 + j) * 8 + g]);
      }
      __syncthreads();  // all reads of X_i done
#pragma unroll
      for (int j = 0; j < JB; ++j) {
        double* xr = X + (rb + gg * 8 + g) * SD_LDX + (nb0 + j) * 8 + 2 * t;
        xr[0] = acc[j][0];
        xr[1] = acc[j][1];
      }
      __syncthreads();
    }
    const int below = rb + 32;
    if (below < np) {  // X_{>i} -= L_{>i,i} X_i: warp w takes 16-row tiles of the rows below
      constexpr int TG = 2;  // row groups of 8 per warp tile (registers: 3 CTAs per SM)
      const int ntiles = (np - below + 8 * TG - 1) / (8 * TG);
      for (int tt = warp; tt < ntiles; tt += 8) {
        const int r0 = below + tt * 8 * TG;
        double acc[TG][NBK][2];
        double al[TG][8];
#pragma unroll
        for (int gg = 0; gg < TG; ++gg) {
          const int r = r0 + gg * 8 + g;
          const bool rok = r < np;
#pragma unroll
          for (int nb = 0; nb < NBK; ++nb) {
            acc[gg][nb][0] = X[r * SD_LDX + nb * 8 + 2 * t];
            acc[gg][nb][1] = X[r * SD_LDX + nb * 8 + 2 * t + 1];
          }
          const double* lr = L + (int64_t)r * ldl + rb;
#pragma unroll
          for (int k4 = 0; k4 < 8; ++k4) al[gg][k4] = (rok && rb + k4 * 4 + t < np) ? lr[k4 * 4 + t] : 0.0;
        }
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
          double bv[NBK];
#pragma unroll
          for (int nb = 0; nb < NBK; ++nb) bv[nb] = -X[(rb + k4 * 4 + t) * SD_LDX + nb * 8 + g];
#pragma unroll
          for (int gg = 0; gg < TG; ++gg)
#pragma unroll
            for (int nb = 0; nb < NBK; ++nb) dmma884(acc[gg][nb][0], acc[gg][nb][1], al[gg][k4], bv[nb]);
        }
#pragma unroll
        for (int gg = 0; gg < TG; ++gg) {
          const int r = r0 + gg * 8 + g;
#pragma unroll
          for (int nb = 0; nb < NBK; ++nb) {
            X[r * SD_LDX + nb * 8 + 2 * t] = acc[gg][nb][0];
            X[r * SD_LDX + nb * 8 + 2 * t + 1] = acc[gg][nb][1];
          }
        }
      }
      __syncthreads();
    }
  }
  if (cok)
    for (int i = rl; i < np; i += RL) a[(d + i) * lda + gc] = X[i * SD_LDX + col];
}

}  // namespace pflu
