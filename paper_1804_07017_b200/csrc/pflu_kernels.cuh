// pflu_kernels.cuh -- sm_100a device kernels for blocked LU with partial pivoting.
//
// Storage: ROW-MAJOR float64, element (i, j) at a[i * lda + j].  Rows are contiguous, so every
// row interchange is a coalesced (128-bit when aligned) row copy and the trailing update's
// operands are "K-contiguous" L21 rows and "N-contiguous" U12 rows.
//
// Kernels (reference functions they replace, pkg/src/panelforge/...):
//   leaf_getf2_kernel   _jit.py:154-187 lu_unb_run  -- cooperative multi-CTA getf2 on a w<=32
//                       column leaf; rows resident in shared memory, one grid barrier per column
//   pivot_plan_kernel   _jit.py:141-151 laswp_run   -- composes b ascending swaps into a gather plan
//   swap_trsm_kernel    _jit.py:141-151 + 104-113   -- laswp (gather/scatter by plan) fused with the
//                       unit-lower triangular solve of the U12 block row
//   trsm_kernel         _jit.py:104-113              -- in-panel unit-lower solve (no swaps)
//   gemm_dmma_kernel    _jit.py:54-80 macro_run      -- C -= A*B on FP64 tensor cores (DMMA 8x8x4)
//   gemm_exact_kernel   _jit.py:54-80 macro_run      -- same update, reference rounding (mul, then sub)
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
// Grid barrier for cooperative launches (sense/generation based, self-resetting).
// bar[0] = arrival count, bar[1] = generation.  All CTAs of the grid must be co-resident
// (guaranteed by cudaLaunchCooperativeKernel).

__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.volatile.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned gen = ld_volatile_u32(bar + 1);
    __threadfence();
    unsigned old = atomicAdd(bar, 1u);
    if (old == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (ld_volatile_u32(bar + 1) == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
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

// ==========================================================================================
// K1: leaf getf2 (cooperative).  Factors storage columns [col0, col0+wact) of rows [r0, m); the
// diagonal of leaf column j is row r0 + j.  CTA q owns rows [r0 + q*R, r0 + (q+1)*R) and keeps their W leaf columns in shared memory.
// Row interchanges are applied across the whole panel column range [pc0, pc1), like
// lu_unb_run's full-width swap (_jit.py:175-179); columns outside the leaf are swapped in
// global memory by the CTA that owns the pivot row.
// Slots (global, double-buffered by column parity): per CTA (W + 2) doubles = candidate row,
// key, row index; plus one diagonal-row entry.

struct LeafArgs {
  double* a;
  int64_t lda, m;
  int64_t r0;                   // diagonal row of the leaf's first column
  int64_t col0;                 // storage column of the leaf's first column
  int64_t wact;                 // leaf width (<= W)
  int64_t pc0, pc1;             // panel storage-column range swapped across (contains the leaf)
  int64_t R;                    // rows per CTA
  int64_t* piv;                 // global 0-based pivot rows, entries [r0, r0 + wact)
  unsigned long long* info;     // atomicMin of (first zero-pivot column + 1)
  double* slots;                // 2 * (gridDim.x + 1) * (W + 2) doubles
  unsigned* bar;                // grid barrier state (2 words, zero-initialised once)
};

constexpr int LEAF_THREADS = 256;

template <int W>
__global__ void __launch_bounds__(LEAF_THREADS, 1) leaf_getf2_kernel(LeafArgs p) {
  extern __shared__ double leaf_smem[];
  constexpr int LD = W + 1;  // odd stride: conflict-free column walks
  const int tid = threadIdx.x;
  const int q = blockIdx.x;
  const int S = gridDim.x;
  const int64_t rbeg = p.r0 + (int64_t)q * p.R;
  const int64_t rend = min(p.m, rbeg + p.R);
  const int nrows = (int)max((int64_t)0, rend - rbeg);
  const int wact = (int)p.wact;
  double* tile = leaf_smem;                    // [R][LD]
  double* u = leaf_smem + p.R * LD;            // [W] pivot row
  double* dg = u + W;                          // [W] old diagonal row
  __shared__ double red_key[LEAF_THREADS / 32];
  __shared__ long long red_row[LEAF_THREADS / 32];
  __shared__ double s_key;
  __shared__ long long s_row;
  __shared__ int s_win;

  // load own rows
  for (int idx = tid; idx < nrows * wact; idx += LEAF_THREADS) {
    int r = idx / wact, c = idx - r * wact;
    tile[r * LD + c] = p.a[(rbeg + r) * p.lda + p.col0 + c];
  }
  __syncthreads();

  const int64_t kmax = min((int64_t)wact, p.m - p.r0);
  const int slot_stride = W + 2;
  for (int j = 0; j < kmax; ++j) {
    const int64_t c = p.r0 + j;  // diagonal row of leaf column j
    const int par = j & 1;
    double* slot_base = p.slots + (size_t)par * (S + 1) * slot_stride;
    // ---- local argmax over own rows >= c
    double bk = -3.0;
    long long br = LLONG_MAX;
    int64_t r_first = max((int64_t)0, c - rbeg);
    for (int64_t r = r_first + tid; r < nrows; r += LEAF_THREADS) {
      double k = pivot_key(tile[r * LD + j], rbeg + r == c);
      if (key_better(k, rbeg + r, bk, br)) { bk = k; br = rbeg + r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ok = __shfl_xor_sync(0xffffffffu, bk, o);
      long long orr = __shfl_xor_sync(0xffffffffu, br, o);
      if (key_better(ok, orr, bk, br)) { bk = ok; br = orr; }
    }
    if ((tid & 31) == 0) { red_key[tid >> 5] = bk; red_row[tid >> 5] = br; }
    __syncthreads();
    if (tid < 32) {
      bk = tid < LEAF_THREADS / 32 ? red_key[tid] : -3.0;
      br = tid < LEAF_THREADS / 32 ? red_row[tid] : LLONG_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ok = __shfl_xor_sync(0xffffffffu, bk, o);
        long long orr = __shfl_xor_sync(0xffffffffu, br, o);
        if (key_better(ok, orr, bk, br)) { bk = ok; br = orr; }
      }
      if (tid == 0) { s_key = bk; s_row = br; }
    }
    __syncthreads();
    // ---- publish candidate row (+ key, row) and, if owned, the diagonal row
    {
      double* my = slot_base + (size_t)q * slot_stride;
      const long long crow = s_row;
      if (s_key > -2.0) {
        for (int cc = tid; cc < wact; cc += LEAF_THREADS) my[cc] = tile[(crow - rbeg) * LD + cc];
      }
      if (tid == 0) { my[W] = s_key; my[W + 1] = (double)crow; }
      if (c >= rbeg && c < rend) {
        double* dslot = slot_base + (size_t)S * slot_stride;
        for (int cc = tid; cc < wact; cc += LEAF_THREADS) dslot[cc] = tile[(c - rbeg) * LD + cc];
      }
    }
    grid_barrier(p.bar, (unsigned)S);
    // ---- global winner
    {
      bk = -3.0;
      br = LLONG_MAX;
      int wq = -1;
      for (int t = tid; t < S; t += LEAF_THREADS) {
        const double* sl = slot_base + (size_t)t * slot_stride;
        double k = __ldcg(sl + W);
        long long rr = (long long)__ldcg(sl + W + 1);
        if (key_better(k, rr, bk, br)) { bk = k; br = rr; wq = t; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ok = __shfl_xor_sync(0xffffffffu, bk, o);
        long long orr = __shfl_xor_sync(0xffffffffu, br, o);
        int oq = __shfl_xor_sync(0xffffffffu, wq, o);
        if (key_better(ok, orr, bk, br)) { bk = ok; br = orr; wq = oq; }
      }
      if ((tid & 31) == 0) { red_key[tid >> 5] = bk; red_row[tid >> 5] = br; }
      __shared__ int red_q[LEAF_THREADS / 32];
      if ((tid & 31) == 0) red_q[tid >> 5] = wq;
      __syncthreads();
      if (tid == 0) {
        double k0 = red_key[0];
        long long r0 = red_row[0];
        int q0 = red_q[0];
        for (int w = 1; w < LEAF_THREADS / 32; ++w)
          if (key_better(red_key[w], red_row[w], k0, r0)) { k0 = red_key[w]; r0 = red_row[w]; q0 = red_q[w]; }
        s_key = k0; s_row = r0; s_win = q0;
      }
      __syncthreads();
    }
    const double wkey = s_key;
    const long long prow = s_row;
    if (!(wkey > 0.0)) {
      // exactly-zero pivot: info = c + 1, column left untouched (_jit.py:171-174)
      if (q == 0 && tid == 0) {
        p.piv[c] = c;
        atomicMin(p.info, (unsigned long long)(c + 1));
      }
      __syncthreads();
      continue;
    }
    {
      const double* wsl = slot_base + (size_t)s_win * slot_stride;
      for (int cc = tid; cc < wact; cc += LEAF_THREADS) u[cc] = __ldcg(wsl + cc);
      if (prow != c && prow >= rbeg && prow < rend) {
        const double* dslot = slot_base + (size_t)S * slot_stride;
        for (int cc = tid; cc < wact; cc += LEAF_THREADS) dg[cc] = __ldcg(dslot + cc);
      }
      if (q == 0 && tid == 0) p.piv[c] = prow;
    }
    __syncthreads();
    if (prow != c) {
      if (c >= rbeg && c < rend)
        for (int cc = tid; cc < wact; cc += LEAF_THREADS) tile[(c - rbeg) * LD + cc] = u[cc];
      if (prow >= rbeg && prow < rend) {
        for (int cc = tid; cc < wact; cc += LEAF_THREADS) tile[(prow - rbeg) * LD + cc] = dg[cc];
        // full-panel-width swap of the columns outside the leaf (global memory)
        double* r1 = p.a + c * p.lda;
        double* r2 = p.a + prow * p.lda;
        const int64_t nleft = p.col0 - p.pc0;
        const int64_t nright = p.pc1 - (p.col0 + wact);
        for (int64_t cc = tid; cc < nleft + nright; cc += LEAF_THREADS) {
          int64_t col = cc < nleft ? p.pc0 + cc : p.col0 + wact + (cc - nleft);
          double t1 = r1[col], t2 = r2[col];
          r1[col] = t2;
          r2[col] = t1;
        }
      }
      __syncthreads();
    }
    // ---- scale by division (_jit.py:180-182) and rank-1 update, mul then sub (_jit.py:183-186)
    {
      const double pivot = u[j];
      for (int64_t r = max((int64_t)0, c + 1 - rbeg) + tid; r < nrows; r += LEAF_THREADS) {
        double* tr = tile + r * LD;
        double l = __ddiv_rn(tr[j], pivot);
        tr[j] = l;
        for (int cc = j + 1; cc < wact; ++cc) tr[cc] = sub_mul_exact(tr[cc], l, u[cc]);
      }
    }
    __syncthreads();
  }
  // write back own rows
  for (int idx = tid; idx < nrows * wact; idx += LEAF_THREADS) {
    int r = idx / wact, c = idx - r * wact;
    p.a[(rbeg + r) * p.lda + p.col0 + c] = tile[r * LD + c];
  }
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
    int ne_local = 0;
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
    (void)ne_local;
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
  for (int i = rl; i < np; i += RL) {
    const int64_t src = plan[1 + i];
    X[i * TW + col] = cok ? a[src * lda + gc] : 0.0;
  }
  for (int e = rl; e < ne; e += RL) {
    const int64_t src = plan[1 + np + 2 * e + 1];
    E[e * TW + col] = cok ? a[src * lda + gc] : 0.0;
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

template <int VEC>
__global__ void __launch_bounds__(GM_THREADS, 2) gemm_dmma_kernel(GemmArgs p) {
  extern __shared__ __align__(128) double gm_smem[];
  double* sA = gm_smem;                                 // [ST][BM*BK]
  double* sB = gm_smem + GM_ST * GM_BM * GM_BK;         // [ST][BK*BN]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 1, wn = warp & 1;
  int tm, tn;
  tile_coords(blockIdx.x, p.tiles_m, p.tiles_n, tm, tn);
  const int m0 = tm * GM_BM, n0 = tn * GM_BN;
  const int KT = (int)((p.K + GM_BK - 1) / GM_BK);

  // prologue: start the operand pipeline, then seed accumulators from C
#pragma unroll
  for (int s = 0; s < GM_ST - 1; ++s) {
    if (s < KT) gemm_load_stage<VEC>(p, sA + s * GM_BM * GM_BK, sB + s * GM_BK * GM_BN, m0, n0, (int64_t)s * GM_BK, tid);
    cp_async_commit();
  }
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = m0 + wm * 64 + i * 8 + g;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t col = n0 + wn * 32 + j * 8 + 2 * t;
      const double* cp = p.c + row * p.ldc + col;
      if (VEC == 2 && row < p.M && col + 1 < p.N) {
        double2 v = *reinterpret_cast<const double2*>(cp);
        acc[i][j][0] = v.x;
        acc[i][j][1] = v.y;
      } else {
        acc[i][j][0] = (row < p.M && col < p.N) ? cp[0] : 0.0;
        acc[i][j][1] = (row < p.M && col + 1 < p.N) ? cp[1] : 0.0;
      }
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
#pragma unroll
    for (int kk = 0; kk < GM_BK; kk += 4) {
      double af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = wm * 64 + i * 8 + g;
        af[i] = cA[row * GM_BK + ((kk + t) ^ ((g & 3) << 2))];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int col = wn * 32 + j * 8 + g;
        bf[j] = -cB[(kk + t) * GM_BN + (col ^ (t << 2))];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = m0 + wm * 64 + i * 8 + g;
    if (row >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t col = n0 + wn * 32 + j * 8 + 2 * t;
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

}  // namespace pflu
