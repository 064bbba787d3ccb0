// pflu_panel.cuh -- persistent panel factorization (PF) kernel, one launch per panel.
//
// Replaces _factor_panel / lu_unb / _jit.lu_unb_run (factor.py:128-144, 235-250; _jit.py:154-187)
// for an (m - r0) x w panel.  S co-resident CTAs (cooperative launch) each own a contiguous chunk of
// R rows.  The panel is processed in blocks of W columns (right-looking inside the panel):
//
//   for each block J:
//     leaf:   W columns, own rows resident in shared memory; per column one all-to-all exchange of
//             (|pivot candidate|, row, candidate row, diagonal row) through "LL" words in global
//             memory -- 8-byte stores holding 32 payload bits + a 32-bit flag, so a reader polls
//             the word itself and no fence or atomic barrier sits on the per-column critical path
//             (the pattern of NCCL's LL protocol).  Ties go to the smallest row, exactly like the
//             strict '>' scan of _jit.py:163-170.
//     swaps:  the block's row interchanges are applied to the panel's other columns after the leaf
//             (deferred; swaps commute with work on disjoint columns, factor.py:466-468).
//     U:      U_J = L_JJ^-1 * A[J rows, right columns], each CTA redundantly, in registers.
//     update: own rows: A[r, right] -= L[r, J] * U_J  -- DMMA (fast) or multiply-then-subtract
//             in ascending k (exact, = _jit.py:183-186 order).
//
// Exactness: every element still receives its updates in ascending pivot order, scaled by
// division, so exact mode is bitwise equal to lu_unb_run on the panel.
#pragma once
#include "pflu_kernels.cuh"

namespace pflu {

constexpr int PF_THREADS = 256;
constexpr int PF_UCH = 64;  // right-columns chunk of the block update
constexpr size_t PF_MBOX_OFFSET = 2 * 257 * 80 + 512;  // words; after slots + sync words
constexpr size_t PF_LL_WORDS = PF_MBOX_OFFSET + 2 * 256 * 256 * 4;

struct PanelArgs {
  double* a;
  int64_t lda, m;
  int64_t r0;       // diagonal row of panel column 0
  int64_t col0;     // storage column of panel column 0
  int w;            // panel width
  int64_t R;        // rows per CTA
  int64_t* piv;     // global 0-based pivot rows, entries [r0, r0 + min(w, m - r0))
  unsigned long long* info;
  unsigned long long* ll;  // LL exchange words
  unsigned* epoch;         // flag base, advanced by every launch
  int exact;
  unsigned long long* prof;  // optional: per-phase clock64 totals of CTA 0 (tools/ only)
};

#define PF_PROF_MARK(i)                                              \
  do {                                                              \
    if (prof_on) {                                                  \
      long long _t = clock64();                                     \
      prof_acc[i] += _t - prof_t;                                   \
      prof_t = _t;                                                  \
    }                                                               \
  } while (0)

// LL words: high 32 bits = flag, low 32 bits = payload
__device__ __forceinline__ void ll_put(unsigned long long* p, unsigned payload, unsigned flag) {
  unsigned long long v = ((unsigned long long)flag << 32) | payload;
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ll_get(const unsigned long long* p, unsigned flag) {
  unsigned long long v;
  do {
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  } while ((unsigned)(v >> 32) != flag);
  return (unsigned)v;
}
__device__ __forceinline__ void ll_put_d(unsigned long long* p, double x, unsigned flag) {
  long long b = __double_as_longlong(x);
  ll_put(p, (unsigned)b, flag);
  ll_put(p + 1, (unsigned)(b >> 32), flag);
}
__device__ __forceinline__ double ll_get_d(const unsigned long long* p, unsigned flag) {
  unsigned lo = ll_get(p, flag), hi = ll_get(p + 1, flag);
  return __longlong_as_double(((long long)hi << 32) | lo);
}

// 16-byte LL access: two self-validating words per load (each 8-byte half is single-copy atomic)
__device__ __forceinline__ void ll_put2(unsigned long long* p, unsigned a, unsigned b, unsigned flag) {
  unsigned long long v0 = ((unsigned long long)flag << 32) | a, v1 = ((unsigned long long)flag << 32) | b;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(p), "l"(v0), "l"(v1) : "memory");
}
__device__ __forceinline__ void ll_put2_d(unsigned long long* p, double x, unsigned flag) {
  const long long b = __double_as_longlong(x);
  ll_put2(p, (unsigned)b, (unsigned)(b >> 32), flag);
}
__device__ __forceinline__ bool ll_try2(const unsigned long long* p, unsigned flag, unsigned& a, unsigned& b) {
  unsigned long long v0, v1;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(v0), "=l"(v1) : "l"(p) : "memory");
  a = (unsigned)v0;
  b = (unsigned)v1;
  return (unsigned)(v0 >> 32) == flag && (unsigned)(v1 >> 32) == flag;
}
__device__ __forceinline__ double ll_get2_d(const unsigned long long* p, unsigned flag) {
  unsigned a, b;
  while (!ll_try2(p, flag, a, b)) {
  }
  return __longlong_as_double(((long long)b << 32) | a);
}

// grid-wide sync through LL flags (S <= PF_THREADS); fences give release/acquire on data
__device__ __forceinline__ void ll_grid_sync(unsigned long long* sync_words, int S, int q, unsigned flag) {
  __syncthreads();
  if (S > 1) {
    if (threadIdx.x == 0) {
      __threadfence();
      ll_put(sync_words + q, 0u, flag);
    }
    if ((int)threadIdx.x < S) ll_get(sync_words + threadIdx.x, flag);
    __threadfence();
  }
  __syncthreads();
}

template <int W>
struct PanelSmem {
  static constexpr int LD = W + 1;
  static size_t bytes(int64_t R, int w) {
    // tile R x LD, U buffer W x (w - W) (>= W x 8), L_JJ W x W, u / dg W each, plan 4W ints
    const int64_t nright = w > W ? w - W : 8;
    return (size_t)(R * LD + (int64_t)W * nright + W * W + 2 * W) * 8 + 4 * W * 8 + 256;
  }
};

template <int W>
__global__ void __launch_bounds__(PF_THREADS, 1) panel_kernel(PanelArgs p) {
  extern __shared__ __align__(16) double pf_smem[];
  constexpr int LD = W + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = blockIdx.x;
  const int S = gridDim.x;
  const int64_t rbeg = p.r0 + (int64_t)q * p.R;
  const int64_t rend = min(p.m, rbeg + p.R);
  const int nrows = (int)max((int64_t)0, rend - rbeg);
  const int w = p.w;
  const int nright_max = w > W ? w - W : 8;
  double* tile = pf_smem;                                 // [R][LD]
  double* ubuf = tile + p.R * LD;                         // [W][nright_max]  U_J (solved)
  double* ljj = ubuf + (int64_t)W * nright_max;           // [W][W]
  double* u = ljj + W * W;                                // [W]
  double* dg = u + W;                                     // [W]
  long long* plan_row = reinterpret_cast<long long*>(dg + W);  // [2W] slot -> row
  int* plan_src = reinterpret_cast<int*>(plan_row + 2 * W);    // [2W] slot -> source slot
  __shared__ double red_key[PF_THREADS / 32];
  __shared__ long long red_row[PF_THREADS / 32];
  __shared__ int red_q[PF_THREADS / 32];
  __shared__ double red2_key[PF_THREADS / 32];
  __shared__ long long red2_row[PF_THREADS / 32];
  __shared__ double s_key;
  __shared__ long long s_row;
  __shared__ int s_win;
  __shared__ int s_nslots;
  __shared__ long long blk_piv[32];  // pivots of the current block (every CTA knows them)

  const unsigned epoch = *(volatile unsigned*)p.epoch;
  // LL layout: [2 parities][S + 1 records][16 + 2W words], then S sync words
  const int rec = 16 + 2 * W;  // [key line: key, row (16 words = 128 B)][data: 2W words]; 128-B aligned
  const int npar = 2;
  unsigned long long* sync_words = p.ll + (size_t)npar * (S + 1) * rec;
  unsigned long long* mbox = p.ll + PF_MBOX_OFFSET;  // [2][reader 256][writer 256][4 words]
  const bool exact = p.exact != 0;
  const bool prof_on = p.prof != nullptr && tid == 0;
  long long prof_t = clock64();
  long long prof_acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long last_gather_done = clock64();

  int pend_kb = 0, pend_nright = 0, pend_right0 = 0;  // U rows awaiting write-back
  int64_t pend_cJ = 0;
  for (int jb = 0; jb < w; jb += W) {
    const int wb = min(W, w - jb);
    const int64_t cJ = p.r0 + jb;  // diagonal row of the block's first column
    if (pend_kb > 0) {  // previous block's U rows: every CTA finished reading the raw values
      for (int idx = tid; idx < pend_kb * pend_nright; idx += PF_THREADS) {
        const int i = idx / pend_nright, col = idx - i * pend_nright;
        const int64_t r = pend_cJ + i;
        if (r >= rbeg && r < rend) p.a[r * p.lda + p.col0 + pend_right0 + col] = ubuf[idx];
      }
      pend_kb = 0;
      __syncthreads();
    }
    // ---------------- 1. load own rows x block columns
    for (int idx = tid; idx < nrows * W; idx += PF_THREADS) {
      const int r = idx / W, c = idx - r * W;
      tile[r * LD + c] = (c < wb) ? p.a[(rbeg + r) * p.lda + p.col0 + jb + c] : 0.0;
    }
    __syncthreads();
    PF_PROF_MARK(0);
    // ---------------- 2. leaf: columns of the block
    const int kmax = (int)min((int64_t)wb, p.m - cJ);
    for (int j = 0; j < kmax; ++j) {
      const int64_t c = cJ + j;
      const unsigned flag = epoch + (unsigned)(jb + j);
      unsigned long long* slots = p.ll + (size_t)(j & (npar - 1)) * (S + 1) * rec;
      // A: local candidate over own rows >= c
      double bk = -3.0;
      long long br = LLONG_MAX;
      for (int64_t r = max((int64_t)0, c - rbeg) + tid; r < nrows; r += PF_THREADS) {
        const double k = pivot_key(tile[r * LD + j], rbeg + r == c);
        if (key_better(k, rbeg + r, bk, br)) { bk = k; br = rbeg + r; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
        const long long orr = __shfl_xor_sync(0xffffffffu, br, o);
        if (key_better(ok, orr, bk, br)) { bk = ok; br = orr; }
      }
      if (lane == 0) { red_key[warp] = bk; red_row[warp] = br; }
      __syncthreads();
      PF_PROF_MARK(1);
      if (warp == 0) {
        bk = lane < PF_THREADS / 32 ? red_key[lane] : -3.0;
        br = lane < PF_THREADS / 32 ? red_row[lane] : LLONG_MAX;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
          const long long orr = __shfl_xor_sync(0xffffffffu, br, o);
          if (key_better(ok, orr, bk, br)) { bk = ok; br = orr; }
        }
        if (S > 1) {
          // B: publish candidate (key, row, row data) -- data before key is irrelevant: every
          // word carries its own flag
          unsigned long long* my = slots + (size_t)q * rec;
          if (bk > -2.0) {
            const double* trow = tile + (br - rbeg) * LD;
            for (int cc = lane; cc < wb; cc += 32) ll_put2_d(my + 16 + 2 * cc, trow[cc], flag);
          }
          // keys are pushed into every reader's mailbox, so each polled line has a single reader SM
          // (many SMs spinning on one line delay the writer's store by microseconds)
          {
            const long long kb_ = __double_as_longlong(bk);
            const unsigned rowoff = (unsigned)(bk > -2.0 ? br - p.r0 : 0);
            unsigned long long* mb = mbox + (size_t)(j & 1) * 256 * 256 * 4 + (size_t)q * 4;
            for (int t = lane; t < S; t += 32) {
              unsigned long long* e = mb + (size_t)t * 256 * 4;
              ll_put2(e, (unsigned)kb_, (unsigned)(kb_ >> 32), flag);
              ll_put2(e + 2, rowoff, 0u, flag);
            }
          }
        }
        if (lane == 0) { s_key = bk; s_row = br; s_win = q; }
      } else if (warp == 1 && S > 1 && c >= rbeg && c < rend) {
        unsigned long long* dslot = slots + (size_t)S * rec;
        const double* trow = tile + (c - rbeg) * LD;
        for (int cc = lane; cc < wb; cc += 32) ll_put2_d(dslot + 16 + 2 * cc, trow[cc], flag);
      }
      if (S == 1) __syncthreads();  // S > 1: the gather below needs no barrier (own record is polled too)
      const long long gc0 = clock64();
      if (prof_on && q < 32) p.prof[8192 + q * 256 + jb + j] = gc0 - last_gather_done;
      PF_PROF_MARK(2);
      if (prof_on && jb == 0 && j >= 4 && j < 7) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        p.prof[q * 16 + 10 + 2 * (j - 4)] = gt;
      }
      // C: gather all candidates
      if (S > 1) {
        bk = -3.0;
        br = LLONG_MAX;
        int wq = -1;
        if (tid < S) {
          const unsigned long long* sl = mbox + (size_t)(j & 1) * 256 * 256 * 4 + (size_t)q * 256 * 4 + (size_t)tid * 4;
          unsigned k0, k1, r0_, r1_;
          bool ok0 = false, ok1 = false;
          while (!(ok0 && ok1)) {  // both 16-byte loads in flight together
            if (!ok0) ok0 = ll_try2(sl, flag, k0, k1);
            if (!ok1) ok1 = ll_try2(sl + 2, flag, r0_, r1_);
          }
          const double k = __longlong_as_double(((long long)k1 << 32) | k0);
          const long long rr = (long long)r0_ + p.r0;
          if (k > -2.0) { bk = k; br = rr; wq = tid; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
          const long long orr = __shfl_xor_sync(0xffffffffu, br, o);
          const int oq = __shfl_xor_sync(0xffffffffu, wq, o);
          if (key_better(ok, orr, bk, br)) { bk = ok; br = orr; wq = oq; }
        }
        if (lane == 0) { red2_key[warp] = bk; red2_row[warp] = br; red_q[warp] = wq; }
        __syncthreads();
        if (warp == 0) {
          bk = lane < PF_THREADS / 32 ? red2_key[lane] : -3.0;
          br = lane < PF_THREADS / 32 ? red2_row[lane] : LLONG_MAX;
          wq = lane < PF_THREADS / 32 ? red_q[lane] : -1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
            const long long orr = __shfl_xor_sync(0xffffffffu, br, o);
            const int oq = __shfl_xor_sync(0xffffffffu, wq, o);
            if (key_better(ok, orr, bk, br)) { bk = ok; br = orr; wq = oq; }
          }
          if (lane == 0) { s_key = bk; s_row = br; s_win = wq; }
        }
        __syncthreads();
      }
      PF_PROF_MARK(3);
      if (prof_on && q == 0) p.prof[4096 + jb + j] = clock64() - gc0;
      if (prof_on && q < 32) p.prof[16384 + q * 256 + jb + j] = clock64() - gc0;
      last_gather_done = clock64();
      if (prof_on && jb == 0 && j >= 4 && j < 7) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        p.prof[q * 16 + 11 + 2 * (j - 4)] = gt;
      }
      const double wkey = s_key;
      const long long prow = s_row;
      if (!(wkey > 0.0)) {
        // exactly-zero pivot: info = c + 1, column left untouched (_jit.py:171-174)
        if (tid == 0) blk_piv[j] = c;
        if (q == 0 && tid == 0) {
          p.piv[c] = c;
          atomicMin(p.info, (unsigned long long)(c + 1));
        }
        continue;  // s_* are rewritten only after the next __syncthreads
      }
      // D: winner row (and the old diagonal row for the owner of the pivot row)
      if (S > 1) {
        if (warp == 0) {
          const unsigned long long* wsl = slots + (size_t)s_win * rec;
          for (int cc = lane; cc < wb; cc += 32) u[cc] = ll_get2_d(wsl + 16 + 2 * cc, flag);
        } else if (warp == 1 && prow != c && prow >= rbeg && prow < rend) {
          if (c >= rbeg && c < rend) {
            for (int cc = lane; cc < wb; cc += 32) dg[cc] = tile[(c - rbeg) * LD + cc];
          } else {
            const unsigned long long* dsl = slots + (size_t)S * rec;
            for (int cc = lane; cc < wb; cc += 32) dg[cc] = ll_get2_d(dsl + 16 + 2 * cc, flag);
          }
        }
      } else {
        if (warp == 0)
          for (int cc = lane; cc < wb; cc += 32) u[cc] = tile[(prow - rbeg) * LD + cc];
        else if (warp == 1 && prow != c)
          for (int cc = lane; cc < wb; cc += 32) dg[cc] = tile[(c - rbeg) * LD + cc];
      }
      if (tid == 0) blk_piv[j] = prow;
      if (q == 0 && tid == 0) p.piv[c] = prow;
      __syncthreads();
      PF_PROF_MARK(4);
      // E: swap inside the block, scale by division, rank-1 update (mul then sub)
      if (prow != c) {
        if (c >= rbeg && c < rend)
          for (int cc = tid; cc < wb; cc += PF_THREADS) tile[(c - rbeg) * LD + cc] = u[cc];
        if (prow >= rbeg && prow < rend)
          for (int cc = tid; cc < wb; cc += PF_THREADS) tile[(prow - rbeg) * LD + cc] = dg[cc];
        __syncthreads();
      }
      {
        const double pivot = u[j];
        for (int64_t r = max((int64_t)0, c + 1 - rbeg) + tid; r < nrows; r += PF_THREADS) {
          double* tr = tile + r * LD;
          const double l = __ddiv_rn(tr[j], pivot);
          tr[j] = l;
          for (int cc = j + 1; cc < wb; ++cc) tr[cc] = sub_mul_exact(tr[cc], l, u[cc]);
        }
      }
      __syncthreads();
      PF_PROF_MARK(5);
    }
    // ---------------- 3. write back own rows >= cJ of the block
    {
      const int r_first = (int)max((int64_t)0, cJ - rbeg);
      for (int idx = r_first * W + tid; idx < nrows * W; idx += PF_THREADS) {
        const int r = idx / W, cc = idx - r * W;
        if (cc < wb) p.a[(rbeg + r) * p.lda + p.col0 + jb + cc] = tile[r * LD + cc];
      }
    }
    const unsigned sflag = epoch + (unsigned)w + 2u * (unsigned)(jb / W);
    __syncthreads();  // blk_piv complete; no grid sync needed: the swaps below touch only columns
                      // outside this block, which no CTA reads or writes during the leaf
    PF_PROF_MARK(6);
    const int kb = kmax;  // pivots of this block
    const int nother = w - wb;
    // ---------------- 4. deferred swaps of this block on the panel's other columns
    if (nother > 0 && kb > 0) {
      if (tid == 0) {
        // slots: 0..kb-1 = rows cJ + i; extra slots for pivot rows >= cJ + kb (first occurrence)
        int ns = kb;
        for (int i = 0; i < kb; ++i) plan_row[i] = cJ + i;
        for (int i = 0; i < kb; ++i) plan_src[i] = i;
        for (int i = 0; i < kb; ++i) {
          const long long r = blk_piv[i];
          int s;
          if (r < cJ + kb) {
            s = (int)(r - cJ);
          } else {
            s = -1;
            for (int e = kb; e < ns; ++e)
              if (plan_row[e] == r) { s = e; break; }
            if (s < 0) { s = ns++; plan_row[s] = r; plan_src[s] = s; }
          }
          if (s != i) { const int t = plan_src[i]; plan_src[i] = plan_src[s]; plan_src[s] = t; }
        }
        s_nslots = ns;
      }
      __syncthreads();
      const int ns = s_nslots;
      // columns of this CTA (cyclic over the S CTAs), gathered then scattered in batches that
      // fit the U buffer
      const int my_cols = (nother - q + S - 1) / S;
      double* gbuf = ubuf;  // reuse: [ns][batch]
      const int batch = max(1, (W * nright_max) / ns);
      for (int cb = 0; cb < my_cols; cb += batch) {
        const int nb_ = min(batch, my_cols - cb);
        for (int idx = tid; idx < ns * nb_; idx += PF_THREADS) {
          const int s = idx / nb_, ci = cb + idx - (idx / nb_) * nb_;
          const int oc = q + ci * S;
          const int pc = oc < jb ? oc : oc + wb;
          gbuf[idx] = p.a[plan_row[plan_src[s]] * p.lda + p.col0 + pc];
        }
        __syncthreads();
        for (int idx = tid; idx < ns * nb_; idx += PF_THREADS) {
          const int s = idx / nb_, ci = cb + idx - (idx / nb_) * nb_;
          const int oc = q + ci * S;
          const int pc = oc < jb ? oc : oc + wb;
          p.a[plan_row[s] * p.lda + p.col0 + pc] = gbuf[idx];
        }
        __syncthreads();
      }
    }
    ll_grid_sync(sync_words, S, q, sflag + 1u);
    PF_PROF_MARK(7);
    // ---------------- 5. U_J = L_JJ^-1 A[J rows, right] and the block update of own rows
    const int right0 = jb + wb;
    const int nright = w - right0;
    if (nright > 0 && kb > 0) {
      for (int idx = tid; idx < W * W; idx += PF_THREADS) {
        const int r = idx / W, cc = idx - r * W;
        ljj[idx] = (r < kb && cc < kb) ? p.a[(cJ + r) * p.lda + p.col0 + jb + cc] : 0.0;
      }
      __syncthreads();
      for (int col = tid; col < nright; col += PF_THREADS) {
        double x[W];
#pragma unroll
        for (int i = 0; i < W; ++i) x[i] = (i < kb) ? p.a[(cJ + i) * p.lda + p.col0 + right0 + col] : 0.0;
#pragma unroll
        for (int i = 0; i < W; ++i) {
#pragma unroll
          for (int r = i + 1; r < W; ++r) x[r] = sub_mul_exact(x[r], ljj[r * W + i], x[i]);
        }
#pragma unroll
        for (int i = 0; i < W; ++i) ubuf[i * nright + col] = x[i];
      }
      __syncthreads();
      PF_PROF_MARK(8);
      // the owner of the U rows writes them back only after the NEXT grid sync: other CTAs may still
      // be reading the raw rows for their own (redundant) solve
      pend_kb = kb; pend_cJ = cJ; pend_nright = nright; pend_right0 = right0;
      // rows below the block: A[r, right] -= L[r, J] * U_J
      const int64_t ub = max(rbeg, cJ + kb);
      const int nupd = (int)max((int64_t)0, rend - ub);
      const int toff = (int)(ub - rbeg);
      if (!exact) {
        // DMMA: warp w handles 8-row groups w, w+8, ...; 64-column chunks; K = W (zero padded)
        const int ngroups = (nupd + 7) / 8;
        const int g = lane >> 2, t = lane & 3;
        for (int c0 = 0; c0 < nright; c0 += PF_UCH) {
          for (int gi = warp; gi < ngroups; gi += PF_THREADS / 32) {
            const int rl = gi * 8 + g;  // local update row
            const bool rok = rl < nupd;
            double* crow = p.a + (ub + rl) * p.lda + p.col0 + right0;
            double acc[8][2];
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
              const int col = c0 + nb * 8 + 2 * t;
              acc[nb][0] = (rok && col < nright) ? crow[col] : 0.0;
              acc[nb][1] = (rok && col + 1 < nright) ? crow[col + 1] : 0.0;
            }
            const double* arow = tile + (int64_t)(toff + rl) * LD;
#pragma unroll
            for (int k4 = 0; k4 < W; k4 += 4) {
              const double av = rok ? arow[k4 + t] : 0.0;
#pragma unroll
              for (int nb = 0; nb < 8; ++nb) {
                const int col = c0 + nb * 8 + g;
                const double bv = (col < nright) ? -ubuf[(k4 + t) * nright + col] : 0.0;
                dmma884(acc[nb][0], acc[nb][1], av, bv);
              }
            }
            if (rok) {
#pragma unroll
              for (int nb = 0; nb < 8; ++nb) {
                const int col = c0 + nb * 8 + 2 * t;
                if (col < nright) crow[col] = acc[nb][0];
                if (col + 1 < nright) crow[col + 1] = acc[nb][1];
              }
            }
          }
        }
      } else {
        for (int idx = tid; idx < nupd * nright; idx += PF_THREADS) {
          const int rl = idx / nright, col = idx - rl * nright;
          double* cp = p.a + (ub + rl) * p.lda + p.col0 + right0 + col;
          const double* arow = tile + (int64_t)(toff + rl) * LD;
          double acc = *cp;
          for (int k = 0; k < kb; ++k) acc = sub_mul_exact(acc, arow[k], ubuf[k * nright + col]);
          *cp = acc;
        }
      }
    }
    // re-align the CTAs before the next leaf: they leave the update at different times, and a
    // skewed start makes early CTAs spin on lines that late CTAs still have to write
    if (jb + W < w) ll_grid_sync(sync_words, S, q, epoch + (unsigned)w + 2u * (unsigned)((w + W - 1) / W) + 8u + (unsigned)(jb / W));
    __syncthreads();
    PF_PROF_MARK(9);
  }
  if (pend_kb > 0) {  // only reachable if the last block had a right part (it never does)
    ll_grid_sync(sync_words, S, q, epoch + (unsigned)w + 2u * (unsigned)((w + W - 1) / W) + 4u);
    for (int idx = tid; idx < pend_kb * pend_nright; idx += PF_THREADS) {
      const int i = idx / pend_nright, col = idx - i * pend_nright;
      const int64_t r = pend_cJ + i;
      if (r >= rbeg && r < rend) p.a[r * p.lda + p.col0 + pend_right0 + col] = ubuf[idx];
    }
  }
  if (prof_on)
    for (int i = 0; i < 10; ++i) p.prof[q * 16 + i] += prof_acc[i];
  // advance the flag base for the next launch (all CTAs read it at their start)
  if (q == 0 && tid == 0) atomicAdd(p.epoch, (unsigned)(w + 3 * ((w + W - 1) / W) + 16));
}

}  // namespace pflu
