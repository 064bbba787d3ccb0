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
#include <type_traits>

#include "pflu_kernels.cuh"

namespace pflu {

constexpr int PF_THREADS = 256;
constexpr int PF_UCH = 64;  // right-columns chunk of the block update
constexpr int PF_WB = 32;   // super-block width of the two-level in-panel update
constexpr size_t PF_MBOX_OFFSET = 2 * 257 * 80 + 512;  // words; after slots + sync words
constexpr size_t PF_SBOX_OFFSET = PF_MBOX_OFFSET + 2 * 256 * 256 * 4;  // grid-sync mailboxes
constexpr size_t PF_LL_WORDS = PF_SBOX_OFFSET + 256 * 256 * 2;

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
  int resync;                // re-align all CTAs every `resync` columns (0 = never)
  int swcap;                 // cluster kernel: doubles of dedicated row-swap staging (0 = use the L block)
  unsigned* sm_mask;         // optional: every CTA ORs in the bit of its SM (the SM-partitioned look-ahead
                             // reserves these SMs for the panel chain)
};

// key polling: spin this many misses before backing off with __nanosleep (whose granularity is
// coarse, ~1 us: a sleep on the critical path costs a column's worth of time)
constexpr int PF_POLL_SPINS = 64;

// per-phase clock totals (tools/panel_prof.py): compiled in only with -DPFLU_PANEL_PROF (the 16 counters
// cost 32 registers in a kernel that already sits at the 255-register limit)
#ifdef PFLU_PANEL_PROF
#define PF_PROF_MARK(i)                                              \
  do {                                                              \
    if (prof_on) {                                                  \
      long long _t = clock64();                                     \
      prof_acc[i] += _t - prof_t;                                   \
      prof_t = _t;                                                  \
    }                                                               \
  } while (0)
#else
#define PF_PROF_MARK(i) do { } while (0)
#endif

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
// sync words carry a per-launch monotonic counter: "reached" = flag at or past the wanted one, so a
// fast writer that already moved on to the next sync cannot strand a slow reader
__device__ __forceinline__ bool ll_reached2(const unsigned long long* p, unsigned flag) {
  unsigned long long v0, v1;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(v0), "=l"(v1) : "l"(p) : "memory");
  return (int)((unsigned)(v0 >> 32) - flag) >= 0 && (int)((unsigned)(v1 >> 32) - flag) >= 0;
}
__device__ __forceinline__ double ll_get2_d(const unsigned long long* p, unsigned flag, int spins = 1 << 30) {
  unsigned a, b;
  // one-shot reads of data that is normally already visible; after `spins` misses back off (the
  // sleep granularity is coarse: ~1 us)
  for (int s = 0; !ll_try2(p, flag, a, b); ++s)
    if (s >= spins) __nanosleep(128);
  return __longlong_as_double(((long long)b << 32) | a);
}

// Grid-wide sync through per-reader mailboxes: CTA q stores its arrival flag into every reader's
// line (sbox[reader][writer], 16 bytes apart) and polls only its own S entries, so no L2 line is
// spun on by more than one SM (many SMs polling one line delay the writer's store by microseconds).
// Fences give release/acquire semantics for the data written before the sync.
__device__ __forceinline__ void ll_grid_sync(unsigned long long* sbox, int S, int q, unsigned flag) {
  __syncthreads();
  if (S > 1) {
    if (threadIdx.x < 32) {
      __threadfence();
      for (int t = threadIdx.x; t < S; t += 32) ll_put2(sbox + ((size_t)t * 256 + q) * 2, 0u, 0u, flag);
    }
    if ((int)threadIdx.x < S) {
      while (!ll_reached2(sbox + ((size_t)q * 256 + threadIdx.x) * 2, flag)) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Re-alignment of all CTAs without memory ordering (no data is published through it): LL flags only.
__device__ __forceinline__ void ll_grid_align(unsigned long long* sbox, int S, int q, unsigned flag) {
  if (S > 1) {
    if (threadIdx.x < 32) {
      for (int t = threadIdx.x; t < S; t += 32) ll_put2(sbox + ((size_t)t * 256 + q) * 2, 0u, 0u, flag);
      for (int t = threadIdx.x; t < S; t += 32) {
        while (!ll_reached2(sbox + ((size_t)q * 256 + t) * 2, flag)) {
        }
      }
    }
    __syncthreads();
  }
}

// ---- cluster (DSMEM) exchange primitives
constexpr int PF_CL_MAX = 16;  // CTAs per cluster (16 = non-portable size)
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cl_map(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// 16-byte store into a peer CTA's shared memory that completes `bytes` on the peer's mbarrier
__device__ __forceinline__ void cl_put16(uint32_t raddr, unsigned long long x, unsigned long long y, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];\n"
               ::"r"(raddr), "l"(x), "l"(y), "r"(rbar) : "memory");
}
__device__ __forceinline__ void cl_expect(uint32_t bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cl_wait(uint32_t bar, unsigned parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                 "selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  }
}
// The same wait with CTA-scope acquire: enough for data that st.async delivered into THIS CTA's shared
// memory (its complete_tx is what the phase waits for) and for reads of peers' shared memory afterwards
// (DSMEM is not cached); the cluster-scope form above makes ptxas emit CCTL.IVALL (an L1 invalidate,
// hundreds of cycles) after every successful wait.
__device__ __forceinline__ void cl_wait_cta(uint32_t bar, unsigned parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 "selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  }
}
// all threads of all CTAs of the cluster; release/acquire at cluster scope (global data included)
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int W>
struct PanelSmem {
  static constexpr int LD = W + 1;
  static constexpr int KM = W > PF_WB ? W : PF_WB;
  // U of a leaf block (W x rest) or of a super-block (PF_WB x rest), rows padded to ldu(rest)
  __host__ __device__ static int ldu(int ncols) { return (ncols + 15) / 16 * 16 + 4; }
  __host__ __device__ static int64_t ubuf_doubles(int w) {
    const int64_t a = (int64_t)W * ldu(w > W ? w - W : 8), b = (int64_t)PF_WB * ldu(w - PF_WB > 8 ? w - PF_WB : 8);
    return a > b ? a : b;
  }
  static size_t bytes(int64_t R, int w, bool cl = false) {
    // tile R x LD, U buffer, L block KM x KM, u / dg W each, plan 4W ints
    // (+ cluster mode: keys [2][PF_CL_MAX][2], published rows [2][W] x 2, 2 mbarriers, alignment)
    // (v2 exchange: keys [2][PF_CL_MAX][8 slots][2], published rows [2][8 slots][W], diagonal rows [2][W])
    return (size_t)(R * LD + ubuf_doubles(w) + KM * KM + 4 * W) * 8 + 4 * W * 8 + 256 +
           (cl ? (size_t)(32 * PF_CL_MAX + 18 * W + 2 + 2) * 8 : 0);
  }
  // row-swap staging that would make the cluster kernel's deferred swaps a single batch
  static int64_t swap_doubles(int w) { return (int64_t)2 * W * (w > W ? w - W : 1); }
};

// CL = false: S co-resident CTAs exchange through LL words in global memory (any S <= 256).
// CL = true:  the S <= 16 CTAs form one thread-block cluster; candidates and the diagonal row are
//             pushed into every peer's shared memory with st.async completing on the peer's mbarrier
//             (no polling, no L2 round trip), and grid syncs are cluster barriers.
// EX: 0 / 1 = the exact flag compiled in (production since round 2: DMMA mode's in-leaf updates are
// single FMAs; this specialisation exposed the zero-pivot reconvergence hazard fixed below);
// -1 = read at run time from p.exact (-DPFLU_PANEL_EXACT_RUNTIME, the round-1 build).
// V2 (cluster kernel with peers only): the per-column exchange is run by a dedicated warp (warp 0) while
// warps 1..7 own fixed rows; every WORKER WARP pushes its own candidate straight to every peer (no CTA-level
// arg-max, no block barrier inside a column) -- see the V2 leaf below.
// MC (v2 only): the grid is several 16-CTA clusters.  Inside a cluster the exchange is the v2 one; the
// exchange warps then trade their cluster's winner (key, row and the row's data) with the same-rank CTAs of
// the other clusters through LL words in global memory -- one inter-cluster round per column, per-reader
// mailboxes -- and the block-level syncs are the grid kernel's LL barrier over all CTAs.
constexpr size_t PF_MC_MSG = 68;      // LL words per inter-cluster message: key, row word, 32 row elements
constexpr int PF_MC_MAXCL = 8;        // clusters per panel (<= 128 CTAs)
template <int W, bool CL, int EX = -1, bool V2 = false, bool MC = false>
__global__ void __launch_bounds__(PF_THREADS, 1) panel_kernel(PanelArgs p) {
  static_assert(!V2 || CL, "the v2 leaf is a cluster exchange");
  static_assert(!MC || V2, "multi-cluster panels use the v2 leaf");
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
  double* ubuf = tile + p.R * LD;                         // U (solved), ubuf_doubles(w)
  double* ljj = ubuf + PanelSmem<W>::ubuf_doubles(w);     // [KM][KM] unit-lower L block
  double* u = ljj + PanelSmem<W>::KM * PanelSmem<W>::KM;  // [2][W] pivot row (double-buffered)
  double* dg = u + 2 * W;                                 // [2][W] old diagonal row
  long long* plan_row = reinterpret_cast<long long*>(dg + 2 * W);  // [2W] slot -> destination row
  long long* plan_src_row = plan_row + 2 * W;                       // [2W] slot -> source row
  // CL: keys pushed by the peers (16-byte aligned for st.async), own published candidate / diagonal
  // rows (pulled by the peers with DSMEM loads), mbarriers; all double-buffered by exchange parity
  // (offset arithmetic on pf_smem keeps the shared address space: LDS/STS instead of generic accesses)
  double* xkey = pf_smem + ((p.R * LD + PanelSmem<W>::ubuf_doubles(w) + PanelSmem<W>::KM * PanelSmem<W>::KM + 8 * W + 1) & ~(int64_t)1);
  double* pubrow = xkey + (V2 ? 2 * PF_CL_MAX * 8 * 2 : 2 * PF_CL_MAX * 2);  // [2][W] (v2: [2][8 slots][W])
  double* pubdiag = pubrow + (V2 ? 16 * W : 2 * W);                          // [2][W]
  unsigned long long* xbar = reinterpret_cast<unsigned long long*>(pubdiag + 2 * W);  // [2]
  double* swbuf = reinterpret_cast<double*>(xbar + 2);  // CL: p.swcap doubles (may be 0)
  unsigned xs = 0;  // CL: exchanges so far (uniform over the cluster): buffer xs & 1, phase (xs >> 1) & 1
  if constexpr (CL) {
    if (tid == 0) {
      for (int i = 0; i < 2; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(xbar + i)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (S > 1) cl_sync();  // peers may push into this CTA's barriers only once they are initialised
    else __syncthreads();
  }
  __shared__ double red_key[PF_THREADS / 32];
  __shared__ long long red_row[PF_THREADS / 32];
  __shared__ int s_nslots;
  __shared__ long long blk_piv[32];  // pivots of the current block (every CTA knows them)
  __shared__ double s_wkey;          // winner of the next column (written by warp 0)
  __shared__ long long s_wrow;
  __shared__ double s_rpiv2[2];  // v2: reciprocal of the pivot (DMMA mode), per exchange parity
  __shared__ int s_wrow2[2];     // v2: winner row as an offset from p.r0; -1 = no non-zero pivot

  const unsigned epoch = (CL && !MC) ? 0u : *(volatile unsigned*)p.epoch;
  if (p.sm_mask && tid == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;\n" : "=r"(smid));
    atomicOr(p.sm_mask + (smid >> 5), 1u << (smid & 31));
  }
  // LL layout: [2 parities][S + 1 records][16 + 2W words], then S sync words
  const int rec = 16 + 2 * W;  // [key line: key, row (16 words = 128 B)][data: 2W words]; 128-B aligned
  unsigned long long* sync_words = p.ll + PF_SBOX_OFFSET;  // [reader 256][writer 256][2 words]
  unsigned long long* mbox = p.ll + PF_MBOX_OFFSET;  // [2][reader 256][writer 256][4 words]
  const bool exact = EX < 0 ? p.exact != 0 : EX != 0;
  // in-leaf rank-1 updates and the U solve: the reference's rounding (multiply, round, subtract) in
  // exact mode; one FMA in DMMA mode (whose trailing GEMM is an FMA chain anyway)
  auto upd = [&](double x, double l, double u) -> double {
    if constexpr (EX == 0) return fma(-l, u, x);
    else return sub_mul_exact(x, l, u);
  };
  const int g_resync = p.resync;
#ifdef PFLU_PANEL_PROF
  const bool prof_on = p.prof != nullptr && (tid == 0 || (V2 && tid == 32));  // v2: exchange warp + one worker
  long long prof_t = clock64();
  long long prof_acc[16] = {};
#endif

  // grid-sync flags: epoch + w + (running count of syncs in this launch); the sync sequence is the same
  // on every CTA, and the epoch advance below exceeds w + the sync count
  unsigned nsync = 0;
  auto sync_flag = [&]() { return epoch + (unsigned)w + (++nsync); };
  // grid-wide barrier with release/acquire for global memory: a cluster barrier (its release is a
  // MEMBAR.GPU, ~2-5 us) only when the cluster has peers; one CTA needs only __syncthreads
  auto grid_sync = [&]() {
    if constexpr (CL && !MC) {
      if (S > 1) cl_sync();
      else __syncthreads();
    } else {
      ll_grid_sync(sync_words, S, q, sync_flag());
    }
  };
  int pend_kb = 0, pend_nright = 0, pend_right0 = 0, pend_ldu = 0;  // U rows awaiting write-back
  int64_t pend_cJ = 0;
  auto write_pend = [&]() {
    for (int idx = tid; idx < pend_kb * pend_nright; idx += PF_THREADS) {
      const int i = idx / pend_nright, col = idx - i * pend_nright;
      const int64_t r = pend_cJ + i;
      if (r >= rbeg && r < rend) p.a[r * p.lda + p.col0 + pend_right0 + col] = ubuf[i * pend_ldu + col];
    }
    pend_kb = 0;
  };
  for (int jb = 0; jb < w; jb += W) {
    const int wb = min(W, w - jb);
    const int64_t cJ = p.r0 + jb;  // diagonal row of the block's first column
    if (!CL && pend_kb > 0) {  // previous block's U rows: every CTA finished reading the raw values
      write_pend();
      __syncthreads();
    }
    // ---------------- 1. load own rows x block columns
    {
      // 8 loads in flight per thread (the rows are lda apart: latency, not bandwidth, bound)
      constexpr int LB = 8;
      const int tot = nrows * W;
      for (int base = tid; base < tot; base += LB * PF_THREADS) {
        double v[LB];
#pragma unroll
        for (int u = 0; u < LB; ++u) {
          const int idx = base + u * PF_THREADS;
          const int r = idx / W, cc = idx - r * W;
          v[u] = (idx < tot && cc < wb) ? p.a[(rbeg + r) * p.lda + p.col0 + jb + cc] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < LB; ++u) {
          const int idx = base + u * PF_THREADS;
          const int r = idx / W, cc = idx - r * W;
          if (idx < tot) tile[r * LD + cc] = v[u];
        }
      }
    }
    __syncthreads();
    PF_PROF_MARK(0);
    // ---------------- 2. leaf: columns of the block
    // Per column: gather the pivot keys -> read the winner row -> (pass 1) swap-in, scale, update
    // column j+1 while tracking its pivot candidate -> publish the candidate (its row finished by
    // warp 0; the next diagonal row by warp 1) -> (pass 2) remaining columns, overlapping the
    // exchange.  Every row is owned by one thread, so the swap needs no barrier.
    const int kmax = (int)min((int64_t)wb, p.m - cJ);
    if constexpr (!V2) {
    auto cta_best = [&](double& bk, long long& br) {
      warp_best(bk, br);
      PF_PROF_MARK(11);
      if (lane == 0) { red_key[warp] = bk; red_row[warp] = br; }
      __syncthreads();
      PF_PROF_MARK(12);
      constexpr int NW = PF_THREADS / 32;
      bk = lane < NW ? red_key[lane] : -3.0;
      br = lane < NW ? red_row[lane] : LLONG_MAX;
      warp_best(bk, br);
    };
    // publish candidate (key, row, data of tile row br) for column jn; warp 0 only
    auto publish_cand = [&](int jn, double bk, long long br) {
      if constexpr (CL) {
        // the finished candidate row goes to the publish buffer, then one (key, row) st.async per
        // peer; its complete_tx has release semantics at cluster scope, so a peer that saw the key
        // can pull the row
        double* pr = pubrow + (xs & 1) * W;
        if (bk > -2.0)
          for (int cc = lane; cc < wb; cc += 32) pr[cc] = tile[(br - rbeg) * LD + cc];
        __syncwarp();
        if (lane < S)
          cl_put16(cl_map(smem_addr(xkey + ((xs & 1) * PF_CL_MAX + q) * 2), lane),
                   (unsigned long long)__double_as_longlong(bk), (unsigned long long)br,
                   cl_map(smem_addr(xbar + (xs & 1)), lane));
        return;
      }
      const unsigned fl = epoch + (unsigned)(jb + jn);
      unsigned long long* sl = p.ll + (size_t)(jn & 1) * (S + 1) * rec;
      unsigned long long* my = sl + (size_t)q * rec;
      if (bk > -2.0) {
        const double* trow = tile + (br - rbeg) * LD;
        for (int cc = lane; cc < wb; cc += 32) ll_put2_d(my + 16 + 2 * cc, trow[cc], fl);
      }
      const long long kb_ = __double_as_longlong(bk);
      const unsigned rowoff = (unsigned)(bk > -2.0 ? br - p.r0 : 0);
      unsigned long long* mb = mbox + (size_t)(jn & 1) * 256 * 256 * 4 + (size_t)q * 4;
      for (int t = lane; t < S; t += 32) {
        unsigned long long* e = mb + (size_t)t * 256 * 4;
        ll_put2(e, (unsigned)kb_, (unsigned)(kb_ >> 32), fl);
        ll_put2(e + 2, rowoff, 0u, fl);
      }
    };
    auto publish_diag = [&](int jn, long long row) {  // the owner of the next diagonal row, one warp
      if constexpr (CL) {  // warp 0, before it pushes its key: the diagonal row to the publish buffer
        double* pd = pubdiag + (xs & 1) * W;
        for (int cc = lane; cc < wb; cc += 32) pd[cc] = tile[(row - rbeg) * LD + cc];
        return;
      }
      const unsigned fl = epoch + (unsigned)(jb + jn);
      unsigned long long* dsl = p.ll + (size_t)(jn & 1) * (S + 1) * rec + (size_t)S * rec;
      const double* trow = tile + (row - rbeg) * LD;
      for (int cc = lane; cc < wb; cc += 32) ll_put2_d(dsl + 16 + 2 * cc, trow[cc], fl);
    };
    // Warp 0 gathers the winner of column jn: the S keys from this CTA's mailbox, then the winner's
    // row (LL slot, or the tile when this CTA owns it -- finished by warp 0 itself) into u[jn & 1] and,
    // when this CTA owns the winner but not the diagonal row, the old diagonal row into dg[jn & 1]
    // (when it owns both, warp 1 staged that row).  (lk, lr) is this CTA's own candidate.
    auto gather = [&](int jn, double lk, long long lr) {
      const unsigned flag = epoch + (unsigned)(jb + jn);
      const int64_t cn = cJ + jn;
      double bk = -3.0;
      long long br = LLONG_MAX;
      int bq = -1;
      if (CL && S > 1) {
        const uint32_t bar = smem_addr(xbar + (xs & 1));
        if (lane == 0) cl_expect(bar, (unsigned)S * 16u);
        cl_wait(bar, (xs >> 1) & 1u);
        PF_PROF_MARK(13);
        if (lane < S) {
          const double* kk = xkey + ((xs & 1) * PF_CL_MAX + lane) * 2;
          const double k = kk[0];
          const long long rr = __double_as_longlong(kk[1]);
          if (k > -2.0) { bk = k; br = rr; }
        }
        bq = warp_best(bk, br);
        PF_PROF_MARK(14);
      } else if (S > 1) {
        const unsigned long long* mb = mbox + (size_t)(jn & 1) * 256 * 256 * 4 + (size_t)q * 256 * 4;
        for (int t = lane; t < S; t += 32) {
          const unsigned long long* e = mb + (size_t)t * 4;
          unsigned k0, k1, r0_, r1_;
          bool ok0 = false, ok1 = false;
          int spins = 0;
          while (!(ok0 && ok1)) {  // both 16-byte loads in flight together
            if (!ok0) ok0 = ll_try2(e, flag, k0, k1);
            if (!ok1) ok1 = ll_try2(e + 2, flag, r0_, r1_);
            if (!(ok0 && ok1) && ++spins > PF_POLL_SPINS) __nanosleep(32);
          }
          const double k = __longlong_as_double(((long long)k1 << 32) | k0);
          const long long rr = (long long)r0_ + p.r0;
          if (k > -2.0 && key_better(k, rr, bk, br)) { bk = k; br = rr; bq = t; }
        }
        bq = __shfl_sync(0xffffffffu, bq, warp_best(bk, br));
      } else {
        bk = lk; br = lr; bq = q;
      }
      if (bk > 0.0) {
        double* un = u + (jn & 1) * W;
        double* dn = dg + (jn & 1) * W;
        const bool own_p = br >= rbeg && br < rend;
        const bool own_cn = cn >= rbeg && cn < rend;
        const unsigned long long* sl = p.ll + (size_t)(jn & 1) * (S + 1) * rec;
        if (CL && S > 1) {
          // pull the winner row (and, for the winner's owner, the old diagonal row) from the owners'
          // publish buffers; both loads in flight together
          const bool need_d = own_p && br != cn && !own_cn;
          const uint32_t ra = cl_map(smem_addr(pubrow + (xs & 1) * W), bq);
          const uint32_t rd = cl_map(smem_addr(pubdiag + (xs & 1) * W), (int)((cn - p.r0) / p.R));
          if (lane < wb) {
            double x, y = 0.0;
            asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(x) : "r"(ra + 8 * lane) : "memory");
            if (need_d) asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(y) : "r"(rd + 8 * lane) : "memory");
            un[lane] = x;
            if (need_d) dn[lane] = y;
          }
          PF_PROF_MARK(15);
        } else if (!own_p) {
          const unsigned long long* wsl = sl + (size_t)bq * rec;
          for (int cc = lane; cc < wb; cc += 32) un[cc] = ll_get2_d(wsl + 16 + 2 * cc, flag, PF_POLL_SPINS);
        } else {
          for (int cc = lane; cc < wb; cc += 32) un[cc] = tile[(br - rbeg) * LD + cc];
        }
        if (!CL && S > 1 && own_p && br != cn && !own_cn) {
          const unsigned long long* dsl = sl + (size_t)S * rec;
          for (int cc = lane; cc < wb; cc += 32) dn[cc] = ll_get2_d(dsl + 16 + 2 * cc, flag, PF_POLL_SPINS);
        }
      }
      if (lane == 0) { s_wkey = bk; s_wrow = br; }
    };
    // warp 1: the owner of the next diagonal row publishes it and stages it as dg[jn & 1]
    auto stage_diag = [&](int jn, long long row) {
      if (S > 1) publish_diag(jn, row);
      const double* trow = tile + (row - rbeg) * LD;
      double* dn = dg + (jn & 1) * W;
      for (int cc = lane; cc < wb; cc += 32) dn[cc] = trow[cc];
    };
    double ck = -3.0;
    long long cr = LLONG_MAX;
    if (kmax > 0) {  // candidate for the block's first column (the tile is current)
      for (int64_t r = max((int64_t)0, cJ - rbeg) + tid; r < nrows; r += PF_THREADS) {
        const double k = pivot_key(tile[r * LD], rbeg + r == cJ);
        if (key_better(k, rbeg + r, ck, cr)) { ck = k; cr = rbeg + r; }
      }
      cta_best(ck, cr);
      if (warp == 0) {
        if (CL && cJ >= rbeg && cJ < rend) stage_diag(0, cJ);
        if (S > 1) publish_cand(0, ck, cr);
        gather(0, ck, cr);
      } else if (!CL && warp == 1 && cJ >= rbeg && cJ < rend) {
        stage_diag(0, cJ);
      }
      __syncthreads();
      ++xs;
    }
    // Per column j (its winner, row and the old diagonal row are in shared memory):
    //   pass 1 (all warps): swap-in, scale by division, update column j+1, its pivot candidate
    //   warp 0: finish the candidate row, publish it, gather the winner of column j+1
    //   warp 1: finish the next diagonal row, publish and stage it
    //   warps 1..7: pass 2 (the remaining columns), overlapping the exchange
    for (int j = 0; j < kmax; ++j) {
      const int64_t c = cJ + j;
      const double wkey = s_wkey;
      const long long prow = s_wrow;
      double* ucur = u + (j & 1) * W;
      double* dcur = dg + (j & 1) * W;
      const bool nxt = j + 1 < kmax;
      PF_PROF_MARK(3);
      if (tid == 0) blk_piv[j] = (wkey > 0.0) ? prow : c;
      if (q == 0 && tid == 0) {
        p.piv[c] = (wkey > 0.0) ? prow : c;
        if (!(wkey > 0.0)) atomicMin(p.info, (unsigned long long)(c + 1));
      }
      // Thread 0 diverged from its warp just above (piv / info stores).  Reconverge warp 0 explicitly
      // before the warp collectives below: without it, the exact-as-template build let lane 0 reach
      // the zero-pivot branch's cta_best on its own and take its own (key, row) as the CTA's winner
      // (wrong pivot after every zero column; a hang of the grid kernel when CTAs then disagreed).
      // Independent thread scheduling gives no reconvergence guarantee after a divergent branch;
      // __syncwarp() is the documented one (tests/test_gpu_panel_stress.py, tools/panel_hazard.sh).
      __syncwarp();
      if (!(wkey > 0.0)) {
        // exactly-zero pivot: column left untouched (_jit.py:171-174); next candidate from the tile
        ck = -3.0;
        cr = LLONG_MAX;
        if (nxt) {
          for (int64_t r = max((int64_t)0, c + 1 - rbeg) + tid; r < nrows; r += PF_THREADS) {
            const double k = pivot_key(tile[r * LD + j + 1], rbeg + r == c + 1);
            if (key_better(k, rbeg + r, ck, cr)) { ck = k; cr = rbeg + r; }
          }
          cta_best(ck, cr);
          if (warp == 0) {
            if (CL && c + 1 >= rbeg && c + 1 < rend) stage_diag(j + 1, c + 1);
            if (S > 1) publish_cand(j + 1, ck, cr);
            gather(j + 1, ck, cr);
          } else if (!CL && warp == 1 && c + 1 >= rbeg && c + 1 < rend) {
            stage_diag(j + 1, c + 1);
          }
          __syncthreads();
          ++xs;
        }
        continue;
      }
      const bool own_c = c >= rbeg && c < rend;
      if (own_c && prow != c)
        for (int cc = tid; cc < wb; cc += PF_THREADS) tile[(c - rbeg) * LD + cc] = ucur[cc];
      // pass 1: swap-in, scale by division (_jit.py:180-182), column j+1, next candidate
      const double pivot = ucur[j];
      const double uj1 = (j + 1 < wb) ? ucur[j + 1] : 0.0;
      ck = -3.0;
      cr = LLONG_MAX;
      const int64_t p1 = max((int64_t)0, c + 1 - rbeg);  // first row of pass 1
      if (prow != c && prow >= rbeg + p1 && prow < rend) {
        // swap-in of the old diagonal row, by the lanes of the warp whose thread owns row prow
        const int owner = (int)((prow - rbeg - p1) % PF_THREADS);
        if (warp == owner / 32) {
          double* tp = tile + (prow - rbeg) * LD;
          for (int cc = lane; cc < wb; cc += 32) tp[cc] = dcur[cc];
          __syncwarp();
        }
      }
      // DMMA mode scales by the reciprocal (one division per thread); exact mode divides every row
      // (the reference's _jit.py:180-182)
      const double rpiv = EX == 0 ? 1.0 / pivot : 0.0;
      {
        // 32-bit local rows in the hot loop (smaller local row <=> smaller global row)
        const int diag_l = (int)(c + 1 - rbeg);
        int crl = INT_MAX;
        for (int r = (int)p1 + tid; r < nrows; r += PF_THREADS) {
          double* tr = tile + r * LD;
          const double l = EX == 0 ? tr[j] * rpiv : __ddiv_rn(tr[j], pivot);
          tr[j] = l;
          if (j + 1 < wb) {
            const double x = upd(tr[j + 1], l, uj1);
            tr[j + 1] = x;
            if (nxt) {
              const double k = pivot_key(x, r == diag_l);
              if (k > ck || (k == ck && r < crl)) { ck = k; crl = r; }
            }
          }
        }
        if (crl != INT_MAX) cr = rbeg + crl;
      }
      PF_PROF_MARK(10);
      if (nxt) cta_best(ck, cr);
      PF_PROF_MARK(1);
      // the next column's candidate and diagonal rows are finished here by warps 0 / 1 and skipped
      // by pass 2
      const bool cand_own = nxt && ck > -2.0;  // cr is one of this CTA's rows
      const bool diag_own = nxt && c + 1 >= rbeg && c + 1 < rend;
      auto finish_row = [&](long long row) {
        double* tr = tile + (row - rbeg) * LD;
        const double l = tr[j];
        for (int cc = j + 2 + lane; cc < wb; cc += 32) tr[cc] = upd(tr[cc], l, ucur[cc]);
        __syncwarp();
      };
      // cluster: the diagonal row is finished and staged by warp 1 in parallel with warp 0's candidate
      // row; warp 0 waits for it (named barrier 1, 64 threads) before pushing its key, since peers
      // pull the diagonal row once they have seen every key
      const bool diag_split = CL && diag_own && !(cand_own && cr == c + 1);
      if (nxt) {
        if (warp == 0) {
          if (cand_own) finish_row(cr);
          if (CL && diag_own && !diag_split) stage_diag(j + 1, c + 1);  // the candidate is the diagonal row
          if (diag_split) asm volatile("bar.sync 1, 64;\n" ::: "memory");
          if (S > 1) {
            publish_cand(j + 1, ck, cr);
            if (!CL && diag_own && cand_own && cr == c + 1) publish_diag(j + 1, c + 1);
          }
          PF_PROF_MARK(2);
          gather(j + 1, ck, cr);
          PF_PROF_MARK(4);
        } else if (warp == 1 && diag_own && !(cand_own && cr == c + 1)) {
          finish_row(c + 1);
          stage_diag(j + 1, c + 1);
          if (diag_split) asm volatile("bar.arrive 1, 64;\n" ::: "memory");
        }
      }
      // pass 2 (warps 1..7): remaining columns (mul then sub, _jit.py:183-186)
      if (j + 2 < wb && warp > 0) {
        constexpr int NT2 = PF_THREADS - 32;
        const int skip_c = cand_own ? (int)(cr - rbeg) : -1, skip_d = diag_own ? (int)(c + 1 - rbeg) : -1;
        for (int r = (int)max((int64_t)0, c + 1 - rbeg) + (tid - 32); r < nrows; r += NT2) {
          if (r == skip_c || r == skip_d) continue;
          double* tr = tile + r * LD;
          const double l = tr[j];
          // four columns per round with every load issued before the stores (tr and ucur may alias
          // as far as the compiler knows, so it would not reorder them itself)
          int cc = j + 2;
          for (; cc + 3 < wb; cc += 4) {
            const double a0 = tr[cc], a1 = tr[cc + 1], a2 = tr[cc + 2], a3 = tr[cc + 3];
            const double u0 = ucur[cc], u1 = ucur[cc + 1], u2 = ucur[cc + 2], u3 = ucur[cc + 3];
            tr[cc] = upd(a0, l, u0);
            tr[cc + 1] = upd(a1, l, u1);
            tr[cc + 2] = upd(a2, l, u2);
            tr[cc + 3] = upd(a3, l, u3);
          }
          for (; cc < wb; ++cc) tr[cc] = upd(tr[cc], l, ucur[cc]);
        }
      }
      __syncthreads();
      PF_PROF_MARK(5);
      // periodic re-alignment: once CTAs drift apart by a column, early arrivals spin on lines the
      // late ones still have to write and the skew sustains itself
      if (nxt) ++xs;
      if (!CL && g_resync > 0 && nxt && ((j + 1) % g_resync) == 0)
        ll_grid_align(sync_words, S, q, sync_flag());
    }
    } else {
      // ---------------- 2 (v2). leaf with a dedicated exchange warp
      // Warps 1..7 ("workers") own fixed rows of the tile (local row rl -> worker thread rl % 224) through
      // both passes, so nothing inside a column needs a block barrier: per column a worker warp runs pass 1
      // on its rows, takes its OWN candidate (warp arg-max), finishes that row (and the next diagonal row
      // when it owns it), copies it to its publish slot and pushes (key, row) to every peer -- 7 keys per
      // CTA -- then runs pass 2 and waits on named barrier 2 for the winner.  Warp 0 ("exchange") waits for
      // the S x 7 keys, reduces them, pulls the winner row (and the old diagonal row when this CTA owns the
      // winner) from the owners' publish slots, forms the pivot's reciprocal while the pull is in flight,
      // writes (winner, row, 1 / pivot) for the workers and arrives on barrier 2.  Everything is double
      // buffered by exchange parity (xs & 1): a buffer is rewritten two exchanges later, which every peer
      // can only reach after the exchange in between -- i.e. after all readers of the old contents are done.
      constexpr int NWK = PF_THREADS / 32 - 1, NT2 = NWK * 32;
      constexpr unsigned FULL = 0xffffffffu;
      const int base = (int)(rbeg - p.r0);  // row offsets from p.r0 fit 32 bits
      // cluster-local identities (MC: q / S stay the grid-wide CTA index / count)
      int CS = S, qc = q;
      if constexpr (MC) {
        unsigned a_, b_;
        asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(a_));
        asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(b_));
        CS = (int)a_;
        qc = (int)b_;
      }
      const int cid = MC ? q / CS : 0, NC = MC ? S / CS : 1;
      unsigned long long* const mc_mb = p.ll + PF_MBOX_OFFSET;  // MC: [2][128 CTAs][PF_MC_MAXCL][PF_MC_MSG]
      unsigned long long* const mc_dg = p.ll;                   // MC: [2][32] the next diagonal row, LL words
      // Messages, 16 bytes per worker warp: (integer key, ~((row offset from p.r0) << 7 | CTA << 3 | worker
      // slot)); the largest (key, word) tuple is the largest key and, among equal keys, the smallest row.
      if (warp > 0) {
        const int wt = tid - 32, ws = warp - 1;
        auto own_warp = [&](int rl) { return (int)(((unsigned)rl % (unsigned)NT2) >> 5); };
        auto first_row = [&](int p1) { return p1 <= wt ? wt : wt + (int)(((unsigned)(p1 - wt) + NT2 - 1) / NT2) * NT2; };
        // lane t pushes to peer t: its key slot and mbarrier in that peer, per parity
        const int peer = lane < CS ? lane : 0;
        const uint32_t rk0 = cl_map(smem_addr(xkey + ((0 * PF_CL_MAX + qc) * 8 + ws) * 2), peer);
        const uint32_t rk1 = cl_map(smem_addr(xkey + ((1 * PF_CL_MAX + qc) * 8 + ws) * 2), peer);
        const uint32_t rb0 = cl_map(smem_addr(xbar), peer), rb1 = cl_map(smem_addr(xbar + 1), peer);
        // this warp's candidate row crl (key K; none if K == ORD_NONE) and, when the warp owns it, the next
        // diagonal row dl: finished for column j (fin), copied to the publish slots, then the key goes out
        auto publish = [&](unsigned long long K, int crl, int dl, bool fin, int j, const double* ucur) {
          const int buf = xs & 1;
          const bool have = K != ORD_NONE;
          if (have && lane < wb) {
            double* tr = tile + crl * LD;
            double v = tr[lane];
            if (fin && lane >= j + 2) {
              v = upd(v, tr[j], ucur[lane]);
              tr[lane] = v;
            }
            pubrow[(buf * 8 + ws) * W + lane] = v;
          }
          if (dl >= 0 && dl < nrows && own_warp(dl) == ws && lane < wb) {
            double* tr = tile + dl * LD;
            double v = tr[lane];
            if (fin && lane >= j + 2 && !(have && crl == dl)) {
              v = upd(v, tr[j], ucur[lane]);
              tr[lane] = v;
            }
            pubdiag[buf * W + lane] = v;
            if constexpr (MC) ll_put2_d(mc_dg + (buf * 32 + lane) * 2, v, epoch + xs);  // for a winner in another cluster
          }
          __syncwarp();
          if (lane < CS)
            cl_put16(buf ? rk1 : rk0, K,
                     (unsigned long long)(have ? ~((unsigned)(base + crl) << 7 | (unsigned)(qc << 3 | ws)) : 0u),
                     buf ? rb1 : rb0);
          ++xs;
        };
        // candidate of column jn from the current tile (block start, or after a zero pivot); dl = local
        // index of that column's diagonal row
        auto cand_tile = [&](int jn, int dl) {
          unsigned long long K = ORD_NONE;
          unsigned crl = ~0u;
#pragma unroll 1
          for (int r = first_row(max(0, dl)); r < nrows; r += NT2) {
            const unsigned long long k = pivot_key_ord(tile[r * LD + jn], r == dl);
            if (k > K) { K = k; crl = (unsigned)r; }  // rows ascend: strict '>' keeps the smallest row
          }
          {
            unsigned h = (unsigned)(K >> 32), m = (unsigned)K, l = ~crl;
            warp_max96(h, m, l);
            K = ((unsigned long long)h << 32) | m;
            crl = ~l;
          }
          publish(K, (int)crl, dl, false, 0, nullptr);
        };
        const int cl0 = (int)max((int64_t)-(1 << 30), min((int64_t)(1 << 30), cJ - rbeg));  // local row of column 0's diagonal
        if (kmax > 0) cand_tile(0, cl0);
        int r1 = first_row(max(0, min(cl0 + 1, nrows)));  // this thread's first row below the diagonal, kept per column
        for (int j = 0; j < kmax; ++j) {
          PF_PROF_MARK(5);
          __syncwarp();
          asm volatile("bar.sync 2, 256;\n" ::: "memory");
          const int rb = (xs - 1) & 1;
          const double rpiv = s_rpiv2[rb];  // 0 exactly when the column has no pivot (key <= 0)
          const double* ucur = u + rb * W;
          const double* dcur = dg + rb * W;
          const bool nxt = j + 1 < kmax;
          const int cl = cl0 + j;  // local index of the diagonal row (any sign)
          const int prl = s_wrow2[rb] - base;  // local index of the pivot row (>= cl); < 0 marks a zero pivot
          if (s_wrow2[rb] < 0) {               // exactly-zero pivot: column untouched (_jit.py:171-174)
            if (nxt) cand_tile(j + 1, cl + 1);
            continue;
          }
          if (prl != cl) {  // swap: the winner row into the diagonal row, the old diagonal row into the winner's
            if (cl >= 0 && cl < nrows && own_warp(cl) == ws && lane < wb) tile[cl * LD + lane] = ucur[lane];
            if (prl >= 0 && prl < nrows && own_warp(prl) == ws && lane < wb) tile[prl * LD + lane] = dcur[lane];
            __syncwarp();
          }
          const double pivot = ucur[j];
          const double uj1 = (j + 1 < wb) ? ucur[j + 1] : 0.0;
          if (r1 < cl + 1) r1 += NT2;  // the diagonal moves down one row per column
          if (rpiv == 123.456) PF_PROF_MARK(15);  // (forces the result loads before the mark)
          PF_PROF_MARK(3);
          unsigned long long K = ORD_NONE;
          unsigned crl = ~0u;
#pragma unroll 1
          for (int r = r1; r < nrows; r += NT2) {  // pass 1: scale, column j+1, its candidate
            double* tr = tile + r * LD;
            const double l = EX == 0 ? tr[j] * rpiv : __ddiv_rn(tr[j], pivot);
            tr[j] = l;
            if (j + 1 < wb) {
              const double x = upd(tr[j + 1], l, uj1);
              tr[j + 1] = x;
              if (nxt) {
                const unsigned long long k = pivot_key_ord(x, r == cl + 1);
                if (k > K) { K = k; crl = (unsigned)r; }
              }
            }
          }
          int skip_c = -1, skip_d = -1;
          PF_PROF_MARK(10);
          if (nxt) {
            {
              unsigned h = (unsigned)(K >> 32), m = (unsigned)K, l = ~crl;
              warp_max96(h, m, l);
              K = ((unsigned long long)h << 32) | m;
              crl = ~l;
            }
            PF_PROF_MARK(11);
            publish(K, (int)crl, cl + 1, true, j, ucur);
            PF_PROF_MARK(2);
            if (K != ORD_NONE) skip_c = (int)crl;
            if (cl + 1 >= 0 && cl + 1 < nrows && own_warp(cl + 1) == ws) skip_d = cl + 1;
          }
          if (j + 2 < wb) {  // pass 2: the remaining columns of the thread's own rows
#pragma unroll 1
            for (int r = r1; r < nrows; r += NT2) {
              if (r == skip_c || r == skip_d) continue;
              double* tr = tile + r * LD;
              const double l = tr[j];
              int cc = j + 2;
#pragma unroll 1
              for (; cc + 3 < wb; cc += 4) {
                const double a0 = tr[cc], a1 = tr[cc + 1], a2 = tr[cc + 2], a3 = tr[cc + 3];
                const double u0 = ucur[cc], u1 = ucur[cc + 1], u2 = ucur[cc + 2], u3 = ucur[cc + 3];
                tr[cc] = upd(a0, l, u0);
                tr[cc + 1] = upd(a1, l, u1);
                tr[cc + 2] = upd(a2, l, u2);
                tr[cc + 3] = upd(a3, l, u3);
              }
              for (; cc < wb; ++cc) tr[cc] = upd(tr[cc], l, ucur[cc]);
            }
          }
        }
      } else {
        // exchange warp: lane handles peer CTA lane / 2, worker slots 4 * (lane & 1) .. + 3.  One warp runs
        // this chain once per column, so its length in instructions is the panel's per-column latency.
        const int R32 = (int)p.R;
        int qd = jb / R32, rem = jb - qd * R32;  // owner CTA of the diagonal row of column jn, kept incrementally
        const int s0 = (lane & 1) * 4;
        const bool lane_on = (lane >> 1) < CS;
        const uint32_t key_a = smem_addr(xkey + ((lane >> 1) * 8 + s0) * 2);  // + buf * PF_CL_MAX * 128 bytes
        const uint32_t pub_a = smem_addr(pubrow) + 8 * lane, dia_a = smem_addr(pubdiag) + 8 * lane;
        if (kmax > 0 && lane == 0) cl_expect(smem_addr(xbar + (xs & 1)), (unsigned)(CS * NWK) * 16u);
        for (int jn = 0; jn < kmax; ++jn) {
          const int buf = xs & 1;
          PF_PROF_MARK(4);
          cl_wait_cta(smem_addr(xbar + buf), (xs >> 1) & 1u);
          PF_PROF_MARK(13);
          unsigned long long K0 = ORD_NONE, K1 = ORD_NONE, K2 = ORD_NONE, K3 = ORD_NONE, y0 = 0, y1 = 0, y2 = 0, y3 = 0;
          if (lane_on) {
            const uint32_t ka = key_a + buf * (PF_CL_MAX * 8 * 16);
            asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];\n" : "=l"(K0), "=l"(y0) : "r"(ka) : "memory");
            asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];\n" : "=l"(K1), "=l"(y1) : "r"(ka + 16) : "memory");
            asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];\n" : "=l"(K2), "=l"(y2) : "r"(ka + 32) : "memory");
            if (s0 + 3 < NWK) asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];\n" : "=l"(K3), "=l"(y3) : "r"(ka + 48) : "memory");
          }
          unsigned l0 = (unsigned)y0, l1 = (unsigned)y1, l2 = (unsigned)y2, l3 = (unsigned)y3;
          max96(K0, l0, K1, l1);
          max96(K2, l2, K3, l3);
          max96(K0, l0, K2, l2);
          unsigned bh = (unsigned)(K0 >> 32), bm = (unsigned)K0, bl = l0;
          warp_max96(bh, bm, bl);
          PF_PROF_MARK(14);
          double x = 0.0;  // this lane's element of the winner row
          if constexpr (MC) {
            // inter-cluster round: pull this cluster's winner row, send (key, row word, row) to the same-rank
            // CTA of every other cluster, take theirs, keep the best tuple and its row
            const unsigned fl = epoch + xs;
            if ((bh | bm) != 0u && lane < wb) {
              const unsigned c32 = ~bl;
              const uint32_t ra = cl_map(pub_a + (uint32_t)((buf * 8 + (int)(c32 & 7u)) * W * 8), (int)((c32 >> 3) & 15u));
              asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(x) : "r"(ra) : "memory");
            }
            unsigned long long* mb = mc_mb + (size_t)buf * (128 * PF_MC_MAXCL * PF_MC_MSG);
            for (int c2 = 0; c2 < NC; ++c2) {
              if (c2 == cid) continue;
              unsigned long long* e = mb + ((size_t)(c2 * CS + qc) * PF_MC_MAXCL + cid) * PF_MC_MSG;
              if (lane < wb) ll_put2_d(e + 4 + 2 * lane, x, fl);
              if (lane == 0) {
                ll_put2(e, bm, bh, fl);
                ll_put2(e + 2, bl, 0u, fl);
              }
            }
            for (int c2 = 0; c2 < NC; ++c2) {
              if (c2 == cid) continue;
              const unsigned long long* e = mb + ((size_t)q * PF_MC_MAXCL + c2) * PF_MC_MSG;
              unsigned k0 = 0, k1 = 0, l_ = 0, z_ = 0, a_ = 0, b_ = 0;
              bool o0 = false, o1 = false, o2 = lane >= wb;
              while (!(o0 && o1 && o2)) {
                if (!o0) o0 = ll_try2(e, fl, k0, k1);
                if (!o1) o1 = ll_try2(e + 2, fl, l_, z_);
                if (!o2) o2 = ll_try2(e + 4 + 2 * lane, fl, a_, b_);
              }
              const bool better = (k1 > bh) | ((k1 == bh) & ((k0 > bm) | ((k0 == bm) & (l_ > bl))));
              if (better) {
                bh = k1; bm = k0; bl = l_;
                x = __longlong_as_double(((long long)b_ << 32) | a_);
              }
            }
          }
          const unsigned r32 = ~bl;
          const int noff = jb + jn;  // offset of this column's diagonal row from p.r0
          const bool ok = bh > 0x80000000u || (bh == 0x80000000u && bm != 0u);  // key > ORD_ZERO: a non-zero pivot
          const int broff = ok ? (int)(r32 >> 7) : noff;
          if (ok) {
            const int bloc = broff - base;
            const bool need_d = bloc >= 0 && bloc < nrows && broff != noff;
            const uint32_t ra = cl_map(pub_a + (uint32_t)((buf * 8 + (int)(r32 & 7u)) * W * 8), (int)((r32 >> 3) & 15u));
            const bool d_local = !MC || qd / CS == cid;  // the diagonal row's owner sits in this cluster
            const uint32_t rd = cl_map(dia_a + (uint32_t)(buf * W * 8), MC ? (d_local ? qd - cid * CS : 0) : qd);
            double y = 0.0;
            if (lane < wb) {
              if constexpr (!MC) asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(x) : "r"(ra) : "memory");
              if (need_d && d_local) asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(y) : "r"(rd) : "memory");
              if (need_d && !d_local) y = ll_get2_d(mc_dg + (buf * 32 + lane) * 2, epoch + xs);
            }
            // |pivot| is the key: the division runs while the pull is in flight (the empty asm pins it
            // between the loads and the stores of their results)
            double rp = 1.0;
            if constexpr (EX == 0) {
              rp = 1.0 / __longlong_as_double((long long)((((unsigned long long)bh << 32) | bm) & 0x7fffffffffffffffull));
              asm volatile("" : "+d"(rp) : : "memory");
            }
            if (lane < wb) {
              u[buf * W + lane] = x;
              if (need_d) dg[buf * W + lane] = y;
            }
            const double pv = __shfl_sync(FULL, x, jn);
            if (lane == 0) {
              s_rpiv2[buf] = (pv != pv) ? pv : copysign(rp, pv);
              s_wrow2[buf] = broff;
            }
            PF_PROF_MARK(15);
          } else if (lane == 0) {
            s_wrow2[buf] = -1;
          }
          __syncwarp();
          asm volatile("bar.arrive 2, 256;\n" ::: "memory");
          // off the critical path: the next exchange's expectation, the pivot record
          ++xs;
          if (lane == 0) {
            if (jn + 1 < kmax) cl_expect(smem_addr(xbar + (xs & 1)), (unsigned)(CS * NWK) * 16u);
            blk_piv[jn] = p.r0 + broff;
            if (q == 0) {
              p.piv[cJ + jn] = p.r0 + broff;
              if (!ok) atomicMin(p.info, (unsigned long long)(cJ + jn + 1));
            }
          }
          if (++rem == R32) { rem = 0; ++qd; }
        }
      }
    }
    __syncthreads();
    // ---------------- 3. write back own rows >= cJ of the block
    {
      const int r_first = (int)max((int64_t)0, cJ - rbeg);
      for (int idx = r_first * W + tid; idx < nrows * W; idx += PF_THREADS) {
        const int r = idx / W, cc = idx - r * W;
        if (cc < wb) p.a[(rbeg + r) * p.lda + p.col0 + jb + cc] = tile[r * LD + cc];
      }
    }
    __syncthreads();  // blk_piv complete; no grid sync needed: the swaps below touch only columns
                      // outside this block, which no CTA reads or writes during the leaf
    PF_PROF_MARK(6);
    const int kb = kmax;  // pivots of this block
    const int nother = w - wb;
    // ---------------- 4. deferred swaps of this block on the panel's other columns
    if (nother > 0 && kb > 0) {
      if (warp == 0) {
        // block swap plan by one warp (kb <= 32, piv[i] >= cJ + i): g(i) = data in row cJ+i before
        // swap i, resolved by pointer jumping over pt(i) = last earlier swap targeting row cJ+i;
        // top row i then receives g(i) (own pivot) / g(ps(i)) / original row piv[i]; an extra row
        // receives g(last swap into it).  plan_row[s] = destination, plan_src[s] -> source row.
        const long long ri = lane < kb ? blk_piv[lane] : -1;
        int pt = -1, ps = -1, nx = -1;
        for (int i2 = 0; i2 < kb; ++i2) {
          const long long v = __shfl_sync(0xffffffffu, ri, i2);
          if (i2 < lane && v == cJ + lane) pt = i2;
          if (i2 < lane && v == ri) ps = i2;
          if (i2 > lane && v == ri && nx < 0) nx = i2;
        }
        long long gi = pt < 0 ? cJ + lane : -1;
        for (int round = 0; round < 6; ++round) {
          const long long gp = __shfl_sync(0xffffffffu, gi, pt < 0 ? lane : pt);
          const int pp = __shfl_sync(0xffffffffu, pt, pt < 0 ? lane : pt);
          if (gi < 0) {
            if (gp >= 0) gi = gp;
            else pt = pp;
          }
        }
        const long long g_ps = __shfl_sync(0xffffffffu, gi, ps < 0 ? lane : ps);
        long long src = ri == cJ + lane ? gi : (ps >= 0 ? g_ps : ri);
        if (lane < kb) { plan_row[lane] = cJ + lane; plan_src_row[lane] = src; }
        const bool extra = lane < kb && ri >= cJ + kb && nx < 0;
        const unsigned em = __ballot_sync(0xffffffffu, extra);
        if (extra) {
          const int e = kb + __popc(em & ((1u << lane) - 1));
          plan_row[e] = ri;
          plan_src_row[e] = gi;
        }
        if (lane == 0) s_nslots = kb + __popc(em);
      }
      __syncthreads();
      const int ns = s_nslots;
      // columns of this CTA (cyclic over the S CTAs), gathered then scattered in batches that
      // fit the U buffer
      const int my_cols = (nother - q + S - 1) / S;
      // staging [ns][batch]: the U buffer (grid kernel), or the free L-block buffer (cluster kernel,
      // whose U buffer may still hold the previous block's U rows)
      const bool own_buf = CL && p.swcap > PanelSmem<W>::KM * PanelSmem<W>::KM;
      double* gbuf = CL ? (own_buf ? swbuf : ljj) : ubuf;
      const int batch = max(1, (CL ? (own_buf ? p.swcap : PanelSmem<W>::KM * PanelSmem<W>::KM) : W * nright_max) / ns);
      for (int cb = 0; cb < my_cols; cb += batch) {
        const int nb_ = min(batch, my_cols - cb);
        // flattened (slot, column) items, 8 loads in flight per thread; the item's slot and column
        // advance incrementally (one division per batch, none per element)
        constexpr int GB = 8;
        const int tot = ns * nb_;
        const int dq = PF_THREADS / nb_, dr = PF_THREADS - dq * nb_;
        auto pcol = [&](int ci) {
          const int oc = q + (cb + ci) * S;
          return oc < jb ? oc : oc + wb;
        };
        auto step = [&](int& s, int& ci) {
          s += dq;
          ci += dr;
          if (ci >= nb_) { ci -= nb_; ++s; }
        };
        {
          int s = tid / nb_, ci = tid - (tid / nb_) * nb_;
          for (int base = tid; base < tot; base += GB * PF_THREADS) {
            double v[GB];
#pragma unroll
            for (int u = 0; u < GB; ++u) {
              const bool ok = base + u * PF_THREADS < tot;
              v[u] = ok ? p.a[plan_src_row[ok ? s : 0] * p.lda + p.col0 + pcol(ci)] : 0.0;
              step(s, ci);
            }
#pragma unroll
            for (int u = 0; u < GB; ++u)
              if (base + u * PF_THREADS < tot) gbuf[base + u * PF_THREADS] = v[u];
          }
        }
        __syncthreads();
        {
          int s = tid / nb_, ci = tid - (tid / nb_) * nb_;
          for (int idx = tid; idx < tot; idx += PF_THREADS) {
            p.a[plan_row[s] * p.lda + p.col0 + pcol(ci)] = gbuf[idx];
            step(s, ci);
          }
        }
        __syncthreads();
      }
    }
    grid_sync();
    if (CL && pend_kb > 0) {  // the previous block's U rows: every CTA has finished reading the raw values
      write_pend();
      __syncthreads();
    }
    PF_PROF_MARK(7);
    // ---------------- 5. U = L^-1 A[pivot rows, target columns], then the update of own rows below.
    // Two levels: every leaf block updates (K = W) only the rest of its PF_WB-wide super-block;
    // the last block of a super-block then applies the whole super-block (K = PF_WB, L streamed
    // from global memory) to the panel columns beyond it.  Each element still receives its
    // updates in ascending k (exact mode stays bitwise equal to the unblocked order).
    auto solve_update = [&](auto kconst, auto tconst, int64_t crow0, int kcnt, int kcol0, int c_lo, int ncols) {
      constexpr int K = decltype(kconst)::value;
      // U rows padded to ldu = 4 (mod 16) doubles: the four k rows of a DMMA B fragment
      // ((k4 + t) * ldu + col) then sit in four different 32-byte bank groups (conflict free)
      const int ldu = PanelSmem<W>::ldu(ncols);
      constexpr bool a_tile = decltype(tconst)::value;  // L operand from the smem tile (else global)
      for (int idx = tid; idx < K * K; idx += PF_THREADS) {
        const int r = idx / K, cc = idx - r * K;
        ljj[idx] = (r < kcnt && cc < kcnt) ? p.a[(crow0 + r) * p.lda + p.col0 + kcol0 + cc] : 0.0;
      }
      __syncthreads();
      for (int col = tid; col < ncols; col += PF_THREADS) {
        double x[K];
#pragma unroll
        for (int i = 0; i < K; ++i) x[i] = (i < kcnt) ? p.a[(crow0 + i) * p.lda + p.col0 + c_lo + col] : 0.0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
#pragma unroll
          for (int r = i + 1; r < K; ++r) x[r] = upd(x[r], ljj[r * K + i], x[i]);
        }
#pragma unroll
        for (int i = 0; i < K; ++i) ubuf[i * ldu + col] = x[i];
      }
      __syncthreads();
      PF_PROF_MARK(8);
      // the owner of the U rows writes them back only after the NEXT grid sync: other CTAs may still
      // be reading the raw rows for their own (redundant) solve
      pend_kb = kcnt; pend_cJ = crow0; pend_nright = ncols; pend_right0 = c_lo; pend_ldu = ldu;
      // own rows below the pivot rows: A[r, cols] -= L[r, k-block] * U
      const int64_t ub = max(rbeg, crow0 + kcnt);
      const int nupd = (int)max((int64_t)0, rend - ub);
      const int toff = (int)(ub - rbeg);
      auto lval = [&](int rl, int k) -> double {
        if (a_tile) return tile[(int64_t)(toff + rl) * LD + k];
        return k < kcnt ? p.a[(ub + rl) * p.lda + p.col0 + kcol0 + k] : 0.0;
      };
      if (!exact) {
        // DMMA: a warp tile is GR row groups x 64 columns; its C values (and, for L from global
        // memory, its L fragment) are all in flight before the first MMA; K zero padded
        constexpr int GR = 2;  // r06: 4 row groups for the tile operand cost the short panels 1-2% and the tall ones 4-6% (registers)
        const int ngroups = (nupd + 7) / 8;
        const int ntr = (ngroups + GR - 1) / GR;      // 32-row tiles
        const int nch = (ncols + PF_UCH - 1) / PF_UCH;
        const int g = lane >> 2, t = lane & 3;
        for (int wt = warp; wt < ntr * nch; wt += PF_THREADS / 32) {
          const int tr_ = wt / nch, c0 = (wt - tr_ * nch) * PF_UCH;
          double acc[GR][8][2];
#pragma unroll
          for (int gg = 0; gg < GR; ++gg) {
            const int rl = (tr_ * GR + gg) * 8 + g;
            const bool rok = rl < nupd;
            const double* crow = p.a + (ub + rl) * p.lda + p.col0 + c_lo;
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
              const int col = c0 + nb * 8 + 2 * t;
              acc[gg][nb][0] = (rok && col < ncols) ? crow[col] : 0.0;
              acc[gg][nb][1] = (rok && col + 1 < ncols) ? crow[col + 1] : 0.0;
            }
          }
          double areg[a_tile ? 1 : GR][a_tile ? 1 : K / 4];
          if constexpr (!a_tile) {
#pragma unroll
            for (int gg = 0; gg < GR; ++gg) {
              const int rl = (tr_ * GR + gg) * 8 + g;
#pragma unroll
              for (int k4 = 0; k4 < K; k4 += 4) areg[gg][k4 / 4] = rl < nupd ? lval(rl, k4 + t) : 0.0;
            }
          }
#pragma unroll
          for (int k4 = 0; k4 < K; k4 += 4) {
            double bv[8];
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
              const int col = c0 + nb * 8 + g;
              bv[nb] = (col < ncols) ? -ubuf[(k4 + t) * ldu + col] : 0.0;
            }
#pragma unroll
            for (int gg = 0; gg < GR; ++gg) {
              const int rl = (tr_ * GR + gg) * 8 + g;
              double av;
              if constexpr (a_tile) av = rl < nupd ? lval(rl, k4 + t) : 0.0;
              else av = areg[gg][k4 / 4];
#pragma unroll
              for (int nb = 0; nb < 8; ++nb) dmma884(acc[gg][nb][0], acc[gg][nb][1], av, bv[nb]);
            }
          }
#pragma unroll
          for (int gg = 0; gg < GR; ++gg) {
            const int rl = (tr_ * GR + gg) * 8 + g;
            if (rl >= nupd) continue;
            double* crow = p.a + (ub + rl) * p.lda + p.col0 + c_lo;
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
              const int col = c0 + nb * 8 + 2 * t;
              if (col < ncols) crow[col] = acc[gg][nb][0];
              if (col + 1 < ncols) crow[col + 1] = acc[gg][nb][1];
            }
          }
        }
      } else {
        for (int idx = tid; idx < nupd * ncols; idx += PF_THREADS) {
          const int rl = idx / ncols, col = idx - rl * ncols;
          double* cp = p.a + (ub + rl) * p.lda + p.col0 + c_lo + col;
          double acc = *cp;
          for (int k = 0; k < kcnt; ++k) acc = sub_mul_exact(acc, lval(rl, k), ubuf[k * ldu + col]);
          *cp = acc;
        }
      }
    };
    {
      const int sbeg = W >= PF_WB ? jb : (jb / PF_WB) * PF_WB;  // super-block of this leaf block
      const int send = W >= PF_WB ? w : min(w, sbeg + PF_WB);
      const int right0 = jb + wb;
      if (send > right0 && kb > 0)
        solve_update(std::integral_constant<int, W>{}, std::true_type{}, cJ, kb, jb, right0, send - right0);
      if (W < PF_WB && right0 == send && send < w) {
        const int kS = (int)min((int64_t)(send - sbeg), p.m - (p.r0 + sbeg));
        if (kS > 0)
          solve_update(std::integral_constant<int, PF_WB>{}, std::false_type{}, p.r0 + sbeg, kS, sbeg, send, w - send);
      }
    }
    // grid kernel: re-align the CTAs before the next leaf (they leave the update at different
    // times, and a skewed start makes early CTAs spin on lines that late CTAs still have to write);
    // the cluster kernel waits on mbarriers instead of polling and needs no re-alignment
    if (!CL && jb + W < w) grid_sync();
    __syncthreads();
    PF_PROF_MARK(9);
  }
  if (pend_kb > 0) {  // the last super-block's U rows (cluster kernel: also the last leaf block's)
    grid_sync();
    write_pend();
  }
#ifdef PFLU_PANEL_PROF
  if (prof_on)
    for (int i = 0; i < 16; ++i) p.prof[(tid == 0 ? 0 : 4096 + 256) + q * 16 + i] += prof_acc[i];
#endif
  // advance the flag base for the next launch (all CTAs read it at their start)
  if constexpr (CL) {
    if (S > 1) cl_sync();  // no CTA may exit while peers can still push into or read its shared memory
  }
  if constexpr (!CL || MC) {
    if (q == 0 && tid == 0) atomicAdd(p.epoch, (unsigned)(2 * w + 4 * ((w + W - 1) / W) + 32));
  }
}

}  // namespace pflu
