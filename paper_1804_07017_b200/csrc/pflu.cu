// pflu.cu -- host driver and C ABI (include/pflu.h) of libpflu.so.
//
// The k-loop of the reference drivers (dmf_mtb, factor.py:382-412; dmf_la, factor.py:455-515)
// runs here in C++.  The two OpenMP sections of dmf_la (branch_a = deferred left swaps +
// TU_L(k) + PF(k+1), branch_b = TU_R(k), factor.py:490-512) become two CUDA streams:
//   sP (highest priority): TU_L(k) -> PF(k+1) -> pivot plan(k+1)
//   sU (lowest priority):  TU_R(k) -> deferred left swaps(k)
// joined by events instead of the per-iteration barrier of sections_2 (runtime.py:278-303):
//   TU_R(k)            waits PF(k)            (pivots + L21 of step k)
//   TU_L(k) + PF(k+1)  waits TU_R(k-1)        (which updated panel k+1's columns)
// There is no host synchronisation inside the factorization.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pflu.h"
#include "pflu_kernels.cuh"
#include "pflu_panel.cuh"
#include "pflu_gemm.cuh"

namespace pflu {

static thread_local std::string g_err;

static int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(expr)                                                                                 \
  do {                                                                                           \
    cudaError_t _e = (expr);                                                                     \
    if (_e != cudaSuccess)                                                                       \
      return set_err(PFLU_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),     \
                     __FILE__, __LINE__);                                                        \
  } while (0)

#define CKR(expr)                 \
  do {                            \
    int _r = (expr);              \
    if (_r != PFLU_OK) return _r; \
  } while (0)

// ------------------------------------------------------------------------------------------
// per-device context

struct DevCtx {
  bool ready = false;
  int dev = -1;
  int sms = 0;
  size_t smem_optin = 0;
  cudaStream_t sP = nullptr, sU = nullptr;
  cudaStream_t sL = nullptr;                 // deferred left swaps
  std::vector<cudaStream_t> sC;              // trailing-update column-chunk streams
  int64_t* plans = nullptr;                  // per-step pivot plans
  size_t plans_cap = 0;                      // in int64 words
  double* dinv = nullptr;                    // per-step inverted 32x32 diagonal blocks of L11 (fast mode)
  size_t dinv_cap = 0;                       // in doubles
  int64_t* plan[2] = {nullptr, nullptr};
  int64_t* rplan = nullptr;                  // recursive panel: pivot plan of the current split
  double* rinv = nullptr;                    // recursive panel: inverted diagonal blocks of that split
  unsigned long long* info = nullptr;
  unsigned long long* ll = nullptr;  // LL exchange words of the panel kernel
  unsigned* epoch = nullptr;
  std::vector<cudaEvent_t> ev;  // event pool (ordering only)
  std::vector<cudaEvent_t> tev; // timing event pool (tracing)
  std::vector<cudaEvent_t> rev; // row-final events of pflu_getrf's streamed D2H
  cudaStream_t sH = nullptr, sD = nullptr;  // pflu_getrf: H2D + factorization / streamed D2H
  double* hbuf = nullptr;                   // pflu_getrf device copy (grow-only)
  size_t hbuf_cap = 0;
  int64_t* hpiv = nullptr;
  size_t hpiv_cap = 0;
  // SM-partitioned look-ahead (pflu_options.malleable): SMs of the panel kernel, per-step tile queues
  unsigned* sm_mask = nullptr;   // 8 words (device)
  unsigned* rec_mask = nullptr;  // host-side switch: the next panel launch records its SMs here
  int* tile_ctr = nullptr;
  size_t tile_ctr_cap = 0;
  std::vector<cudaEvent_t> swev;  // per step: TU_R(k)'s swap + solve done (the join grid waits on it)
};

static std::atomic<long long> g_launches{0};
static unsigned long long* g_prof = nullptr;  // device buffer for panel-kernel phase clocks (tools only)
static int g_pf_cap = []() { const char* e = getenv("PFLU_PANEL_CAP"); return e ? atoi(e) : 32; }();
static int g_gemm_variant = []() { const char* e = getenv("PFLU_GEMM_VARIANT"); return e ? atoi(e) : 0; }();
static thread_local DevCtx* g_dc = nullptr;  // context of the current call (set by ctx_get)
static int g_leaf = []() { const char* e = getenv("PFLU_LEAF"); return e ? atoi(e) : 0; }();
// cluster panel: max CTAs per cluster (0 = LL kernel only), min rows per CTA, max panel rows
static int g_cluster = []() { const char* e = getenv("PFLU_CLUSTER"); return e ? atoi(e) : 16; }();
static int g_auto_rec_leaf = []() { const char* e = getenv("PFLU_AUTO_REC_LEAF"); return e ? atoi(e) : 128; }();
static int64_t g_auto_rec_minrows = []() { const char* e = getenv("PFLU_AUTO_REC_MINROWS"); return e ? atoll(e) : 4096; }();
static int64_t g_mc_minrows = []() { const char* e = getenv("PFLU_MC_MINROWS"); return e ? atoll(e) : 8192; }();
static int64_t g_mc_rows = []() { const char* e = getenv("PFLU_MC_ROWS"); return e ? std::max<int64_t>(512, atoll(e)) : 8192; }();  // rows per cluster
// the kernel of tall panels that sit alone on the critical path (depth 0, multi-rank owners): 4 = multi-cluster
// (falls back to the grid kernel where it does not fit), 1 = the cooperative grid kernel
static int64_t g_la_tall_rows = []() { const char* e = getenv("PFLU_LA_TALL_ROWS"); return e ? atoll(e) : (int64_t)1 << 40; }();
static int g_mc_adapt = []() { const char* e = getenv("PFLU_MC_ADAPT"); return e ? atoi(e) : 1; }();
static int g_first_block = []() { const char* e = getenv("PFLU_FIRST_BLOCK"); return e ? atoi(e) : 0; }();
static int g_tall_kernel = []() { const char* e = getenv("PFLU_TALL_KERNEL"); return e ? atoi(e) : 4; }();
// Clusters for a multi-rank owner's tall panel (multi-cluster kernel).  While the rank's own share of the
// trailing update of this step outlasts the panel + TU_L, the step is bound by SM time, not by the chain:
// two clusters (32 SMs, ~20% slower panel, 40% less SM time) leave more of the GPU to the update; once the
// chain is the longer one, every cluster the device holds (8-rank model, C4: 175.2 -> 168 ms).  Times in ms:
// the update at the in-step DMMA rate, the panel from the measured 0.63 + 1.65e-5 * rows (4 clusters).
static int tall_panel_ctas(int64_t rows, int64_t local_cols, int64_t bw) {
  const double t_upd = 2.0 * (double)rows * (double)local_cols * (double)bw / 33.0e12 * 1e3;
  const double t_chain = 0.83 + 1.65e-5 * (double)rows;
  return t_upd > t_chain ? 2 * PF_CL_MAX : 0;
}
static int g_mc_maxcl = []() { const char* e = getenv("PFLU_MC_MAXCL"); return e ? std::min(PF_MC_MAXCL, std::max(2, atoi(e))) : 4; }();
#ifdef PFLU_PANEL_EXACT_RUNTIME
static int g_pf_v2 = 0;  // the round-1 runtime-flag build has only the v1 kernels
#else
static int g_pf_v2 = []() { const char* e = getenv("PFLU_PANEL_V2"); return e ? atoi(e) : 1; }();
#endif
static int g_cl_minrows = []() { const char* e = getenv("PFLU_CL_MINROWS"); return e ? std::max(1, atoi(e)) : 32; }();
static int64_t g_cl_rows = []() { const char* e = getenv("PFLU_CL_ROWS"); return e ? atoll(e) : (int64_t)1 << 40; }();
static int g_trsm_dmma = []() { const char* e = getenv("PFLU_TRSM_DMMA"); return e ? atoi(e) : 1; }();
static int64_t g_grid_rows = []() { const char* e = getenv("PFLU_GRID_ROWS"); return e ? atoll(e) : 8192; }();
static int g_resync = []() { const char* e = getenv("PFLU_PANEL_RESYNC"); return e ? atoi(e) : 4; }();
static int g_chunks_env = []() { const char* e = getenv("PFLU_CHUNKS"); return e ? atoi(e) : 0; }();  // 0: by size (getrf_async)
static int g_tur_grid = []() { const char* e = getenv("PFLU_TUR_GRID"); return e ? atoi(e) : 0; }();
// recursive panel (panel_kernel 3): leaf width and leaf kernel (0 auto, 1 grid, 2 cluster)
static int g_rec_leaf = []() { const char* e = getenv("PFLU_REC_LEAF"); return e ? atoi(e) : 32; }();
static int g_rec_leafk = []() { const char* e = getenv("PFLU_REC_LEAFK"); return e ? atoi(e) : 0; }();
// force the panel kernel of every PF step of getrf (-1 = the schedule's own choice)
static int g_pf_force = []() { const char* e = getenv("PFLU_PF_KERNEL"); return e ? atoi(e) : -1; }();
// scaling model (tools/emu_scaling.py): emulate one rank of a P-GPU 1-D block-cyclic run whose
// rank owns EVERY panel (the per-step critical path: TU_L + PF) but only 1/P of each trailing update
static int g_emu_ranks = []() { const char* e = getenv("PFLU_EMU_RANKS"); return e ? atoi(e) : 0; }();
// look-ahead-1 schedule with the swap+TRSM of every step overlapped with the previous GEMM
// DMMA swap+TRSM strip width for blocks of <= 256 rows (32 or 16 columns per CTA)
static int g_swap_bn = []() { const char* e = getenv("PFLU_SWAP_BN"); return e ? atoi(e) : 16; }();  // C4: 16 -> 764.5, 32 -> 769.2 ms
// strip width of the pure row-permutation kernel (deferred left swaps): 16 or 32 columns
static int g_lswap_tw = []() { const char* e = getenv("PFLU_LSWAP_TW"); return e ? atoi(e) : 16; }();
static int g_emu_grid_ranks = []() { const char* e = getenv("PFLU_EMU_GRID_RANKS"); return e ? atoi(e) : 4; }();
static int g_tur_split = []() { const char* e = getenv("PFLU_TUR_SPLIT"); return e ? atoi(e) : 0; }();

// Trace of one factorization: pairs of timing events around PF / TU / TU_L / TU_R / GEMM.
static std::atomic<unsigned> g_trace_mask{~0u};  // record kinds a trace collects (pflu_set_trace_mask)
struct Tracer {
  DevCtx* c = nullptr;
  bool on = false;
  size_t used = 0;
  cudaEvent_t t0 = nullptr;
  struct Rec { int label, k; cudaEvent_t e0, e1; double flop; };
  std::vector<Rec> recs;
  int ev(cudaEvent_t* out) {
    if (used == c->tev.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c->tev.push_back(e);
    }
    *out = c->tev[used++];
    return PFLU_OK;
  }
  int start(cudaStream_t st) {
    if (!on) return PFLU_OK;
    CKR(ev(&t0));
    CK(cudaEventRecord(t0, st));
    return PFLU_OK;
  }
  int begin(int label, int k, cudaStream_t st, int* idx, double flop = 0.0) {
    *idx = -1;
    if (!on || !((g_trace_mask.load(std::memory_order_relaxed) >> label) & 1u)) return PFLU_OK;
    Rec r{label, k, nullptr, nullptr, flop};
    CKR(ev(&r.e0));
    CKR(ev(&r.e1));
    CK(cudaEventRecord(r.e0, st));
    recs.push_back(r);
    *idx = (int)recs.size() - 1;
    return PFLU_OK;
  }
  int end(int idx, cudaStream_t st) {
    if (!on || idx < 0) return PFLU_OK;
    CK(cudaEventRecord(recs[idx].e1, st));
    return PFLU_OK;
  }
  int collect(pflu_trace_event* out, int cap, int* len) {
    int n = 0;
    if (on && out) {
      for (const Rec& r : recs) {
        if (n >= cap) break;
        float a = 0.f, b = 0.f;
        CK(cudaEventElapsedTime(&a, t0, r.e0));
        CK(cudaEventElapsedTime(&b, t0, r.e1));
        out[n].label = r.label; out[n].k = r.k; out[n].start_ms = a; out[n].end_ms = b; out[n].flop = r.flop;
        ++n;
      }
    }
    if (len) *len = n;
    return PFLU_OK;
  }
};

static std::mutex g_mu;      // one public call at a time (the library is not re-entrant)
static std::mutex g_ctx_mu;  // device-context creation (pflu_getrf_mg drives devices from several threads)
static DevCtx g_ctx[64];

static constexpr int PF_MAX_CTAS = PF_THREADS;

#ifndef PFLU_PANEL_EXACT_RUNTIME
// the exact flag compiled into the panel kernel (see panel_kernel's EX)
template <int EX>
static const void* pf_fn_ex(int W, bool cl, bool v2, bool mc = false) {
  if (cl && v2 && mc) return W == 8 ? (const void*)panel_kernel<8, true, EX, true, true> : W == 16 ? (const void*)panel_kernel<16, true, EX, true, true>
                                                                                         : (const void*)panel_kernel<32, true, EX, true, true>;
  if (cl && v2) return W == 8 ? (const void*)panel_kernel<8, true, EX, true> : W == 16 ? (const void*)panel_kernel<16, true, EX, true>
                                                                                   : (const void*)panel_kernel<32, true, EX, true>;
  if (cl) return W == 8 ? (const void*)panel_kernel<8, true, EX> : W == 16 ? (const void*)panel_kernel<16, true, EX>
                                                                           : (const void*)panel_kernel<32, true, EX>;
  return W == 8 ? (const void*)panel_kernel<8, false, EX> : W == 16 ? (const void*)panel_kernel<16, false, EX>
                                                                    : (const void*)panel_kernel<32, false, EX>;
}
static const void* pf_fn(int W, bool cl, bool exact = false, bool v2 = false, bool mc = false) {
  return exact ? pf_fn_ex<1>(W, cl, v2, mc) : pf_fn_ex<0>(W, cl, v2, mc);
}
#else
static const void* pf_fn(int W, bool cl, bool exact = false, bool v2 = false, bool mc = false) {
  (void)exact;
  (void)v2;
  (void)mc;
  if (cl) return W == 8 ? (const void*)panel_kernel<8, true> : W == 16 ? (const void*)panel_kernel<16, true>
                                                                       : (const void*)panel_kernel<32, true>;
  return W == 8 ? (const void*)panel_kernel<8, false> : W == 16 ? (const void*)panel_kernel<16, false>
                                                                : (const void*)panel_kernel<32, false>;
}
#endif
static constexpr int MAX_CHUNKS = 8;
static constexpr size_t LL_WORDS = PF_LL_WORDS;

static int ctx_get(DevCtx** out) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return set_err(PFLU_ERR_UNSUPPORTED, "device index %d", dev);
  DevCtx& c = g_ctx[dev];
  std::unique_lock<std::mutex> init_lock(g_ctx_mu, std::defer_lock);
  if (!c.ready) init_lock.lock();  // several host threads may drive one device (pflu_getrf_mg)
  if (!c.ready) {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10)
      return set_err(PFLU_ERR_UNSUPPORTED, "libpflu is built for sm_100a (B200); device %d is sm_%d%d",
                     dev, prop.major, prop.minor);
    c.dev = dev;
    c.sms = prop.multiProcessorCount;
    c.smem_optin = prop.sharedMemPerBlockOptin;
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&c.sP, cudaStreamNonBlocking, hi));
    CK(cudaStreamCreateWithPriority(&c.sU, cudaStreamNonBlocking, lo));
    CK(cudaStreamCreateWithPriority(&c.sL, cudaStreamNonBlocking, lo));
    CK(cudaStreamCreateWithPriority(&c.sH, cudaStreamNonBlocking, lo));
    CK(cudaStreamCreateWithPriority(&c.sD, cudaStreamNonBlocking, lo));
    c.sC.resize(MAX_CHUNKS);
    for (auto& s : c.sC) CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, lo));
    CK(cudaMalloc(&c.plan[0], sizeof(int64_t) * (1 + 3 * PLAN_MAX)));
    CK(cudaMalloc(&c.plan[1], sizeof(int64_t) * (1 + 3 * PLAN_MAX)));
    CK(cudaMalloc(&c.rplan, sizeof(int64_t) * (1 + 3 * PLAN_MAX)));
    CK(cudaMalloc(&c.rinv, sizeof(double) * 1024 * (PLAN_MAX / 32)));
    CK(cudaMalloc(&c.info, 64));
    CK(cudaMalloc(&c.ll, sizeof(unsigned long long) * LL_WORDS));
    CK(cudaMemset(c.ll, 0, sizeof(unsigned long long) * LL_WORDS));
    CK(cudaMalloc(&c.epoch, 64));
    {
      unsigned one = 1;
      CK(cudaMemcpy(c.epoch, &one, sizeof(one), cudaMemcpyHostToDevice));
    }
    // kernel attributes (dynamic shared memory beyond 48 KB; the limit excludes static smem)
    auto allow = [&](const void* fn) -> cudaError_t {
      cudaFuncAttributes fa;
      cudaError_t e = cudaFuncGetAttributes(&fa, fn);
      if (e != cudaSuccess) return e;
      return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(c.smem_optin - fa.sharedSizeBytes));
    };
    for (int W : {8, 16, 32})
      for (bool cl : {false, true})
        for (bool ex : {false, true})
          for (bool v2 : {false, true}) {
            if (v2 && !cl) continue;
            CK(allow(pf_fn(W, cl, ex, v2)));
            if (cl) CK(cudaFuncSetAttribute(pf_fn(W, cl, ex, v2), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
#ifndef PFLU_PANEL_EXACT_RUNTIME
            if (v2) {
              CK(allow(pf_fn(W, cl, ex, v2, true)));
              CK(cudaFuncSetAttribute(pf_fn(W, cl, ex, v2, true), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            }
#endif
          }
    CK(allow((const void*)swap_trsm_kernel<8>));
    CK(allow((const void*)swap_trsm_dmma_kernel<256, 32>));
    CK(allow((const void*)swap_trsm_dmma_kernel<256, 16>));
    CK(allow((const void*)swap_trsm_dmma_kernel<512, 16>));
    CK(allow((const void*)swap_trsm_kernel<16>));
    CK(allow((const void*)swap_trsm_kernel<32>));
    CK(allow((const void*)trsm_kernel<8>));
    CK(allow((const void*)trsm_kernel<16>));
    CK(allow((const void*)trsm_kernel<32>));
    CK(allow((const void*)gemm_exact_kernel<1>));
    CK(allow((const void*)gemm_exact_kernel<2>));
    c.ready = true;
  }
  *out = &c;
  g_dc = &c;
  return PFLU_OK;
}

static int ctx_events(DevCtx& c, size_t n) {
  while (c.ev.size() < n) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.ev.push_back(e);
  }
  return PFLU_OK;
}

static inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ------------------------------------------------------------------------------------------
// kernel launchers (all asynchronous on `st`)

template <class C>
static int launch_gemm_t(const GemmArgs& p0, bool v2, cudaStream_t st) {
  static bool attr_dev[64] = {};
  int attr_d = 0;
  CK(cudaGetDevice(&attr_d));
  bool& attr = attr_dev[attr_d & 63];
  if (!attr) {
    CK(cudaFuncSetAttribute(gemm_dmma_t<C, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    CK(cudaFuncSetAttribute(gemm_dmma_t<C, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  GemmArgs p = p0;
  const int64_t tm = (p.M + C::BM - 1) / C::BM, tn = (p.N + C::BN - 1) / C::BN;
  if (tm * tn > INT_MAX) return set_err(PFLU_ERR_UNSUPPORTED, "gemm grid too large");
  p.tiles_m = (int)tm;
  p.tiles_n = (int)tn;
  if (v2) gemm_dmma_t<C, 2><<<(unsigned)(tm * tn), C::THREADS, C::SMEM, st>>>(p);
  else gemm_dmma_t<C, 1><<<(unsigned)(tm * tn), C::THREADS, C::SMEM, st>>>(p);
  return PFLU_OK;
}

// persistent launch: at most `ctas` CTAs (0 = SMs x resident CTAs per SM)
template <class C, bool PREF = false>
static int launch_gemm_p(DevCtx& dc, const GemmArgs& p0, bool v2, int ctas, cudaStream_t st) {
  static bool attr_dev[64] = {};
  int attr_d = 0;
  CK(cudaGetDevice(&attr_d));
  bool& attr = attr_dev[attr_d & 63];
  if (!attr) {
    CK(cudaFuncSetAttribute(gemm_dmma_persistent<C, 1, PREF>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    CK(cudaFuncSetAttribute(gemm_dmma_persistent<C, 2, PREF>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  GemmArgs p = p0;
  const int64_t tm = (p.M + C::BM - 1) / C::BM, tn = (p.N + C::BN - 1) / C::BN;
  if (tm * tn > INT_MAX) return set_err(PFLU_ERR_UNSUPPORTED, "gemm grid too large");
  p.tiles_m = (int)tm;
  p.tiles_n = (int)tn;
  int grid = ctas > 0 ? ctas : dc.sms * C::MINB;
  grid = (int)std::min<int64_t>(grid, tm * tn);
  if (v2) gemm_dmma_persistent<C, 2, PREF><<<grid, C::THREADS, C::SMEM, st>>>(p);
  else gemm_dmma_persistent<C, 1, PREF><<<grid, C::THREADS, C::SMEM, st>>>(p);
  return PFLU_OK;
}

// TMA-fed GEMM: tensor maps of the A (M x K) and B (K x N) views, encoded on the host per launch
// (cuTensorMapEncodeTiled through the runtime's driver entry point; no libcuda link dependency).
typedef CUresult (*PfnEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PfnEncodeTiled tma_encoder() {
  static PfnEncodeTiled fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PfnEncodeTiled)f;
    else
      cudaGetLastError();
  }
  return fn;
}
static int g_gemm_tma = []() { const char* e = getenv("PFLU_GEMM_TMA"); return e ? atoi(e) : 0; }();

// returns PFLU_OK with *done = false when the views do not meet TMA's alignment rules
template <class C>
static int launch_gemm_tma(const GemmArgs& p, cudaStream_t st, bool* done) {
  *done = false;
  PfnEncodeTiled enc = tma_encoder();
  if (!enc) return PFLU_OK;
  if ((reinterpret_cast<uintptr_t>(p.a) & 15) || (reinterpret_cast<uintptr_t>(p.b) & 15) ||
      (reinterpret_cast<uintptr_t>(p.c) & 15) || (p.lda & 1) || (p.ldb & 1) || (p.ldc & 1) ||
      p.M >= (int64_t)1 << 31 || p.N >= (int64_t)1 << 31 || p.K >= (int64_t)1 << 31)
    return PFLU_OK;
  static bool attr_dev[64] = {};
  int attr_d = 0;
  CK(cudaGetDevice(&attr_d));
  bool& attr = attr_dev[attr_d & 63];
  if (!attr) {
    CK(cudaFuncSetAttribute(gemm_dmma_tma<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, TmaCfg<C>::SMEM));
    attr = true;
  }
  CUtensorMap ta, tb;
  const cuuint32_t es[2] = {1, 1};
  const cuuint64_t da[2] = {(cuuint64_t)p.K, (cuuint64_t)p.M}, sa[1] = {(cuuint64_t)p.lda * 8};
  const cuuint32_t ba[2] = {8, (cuuint32_t)C::BM};
  CUresult r = enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p.a), da, sa, ba, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(PFLU_ERR_CUDA, "cuTensorMapEncodeTiled(A) failed: %d", (int)r);
  const cuuint64_t db[2] = {(cuuint64_t)p.N, (cuuint64_t)p.K}, sb[1] = {(cuuint64_t)p.ldb * 8};
  const cuuint32_t bb[2] = {8, (cuuint32_t)C::BK};
  r = enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p.b), db, sb, bb, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(PFLU_ERR_CUDA, "cuTensorMapEncodeTiled(B) failed: %d", (int)r);
  const int64_t tm = (p.M + C::BM - 1) / C::BM, tn = (p.N + C::BN - 1) / C::BN;
  if (tm * tn > INT_MAX) return set_err(PFLU_ERR_UNSUPPORTED, "gemm grid too large");
  TmaGemmArgs q;
  q.c = p.c; q.ldc = p.ldc; q.M = p.M; q.N = p.N; q.K = p.K;
  q.tiles_m = (int)tm; q.tiles_n = (int)tn;
  gemm_dmma_tma<C><<<(unsigned)(tm * tn), C::THREADS, TmaCfg<C>::SMEM, st>>>(ta, tb, q);
  *done = true;
  return PFLU_OK;
}

// warp-specialised TMA GEMM (gemm_dmma_ws); same tensor maps as launch_gemm_tma with the box
// height of the WS tile.  *done = false when the views do not meet TMA's alignment rules.
template <class C>
static int launch_gemm_ws(const GemmArgs& p, cudaStream_t st, bool* done) {
  *done = false;
  PfnEncodeTiled enc = tma_encoder();
  if (!enc) return PFLU_OK;
  if ((reinterpret_cast<uintptr_t>(p.a) & 15) || (reinterpret_cast<uintptr_t>(p.b) & 15) ||
      (reinterpret_cast<uintptr_t>(p.c) & 15) || (p.lda & 1) || (p.ldb & 1) || (p.ldc & 1) ||
      p.M >= (int64_t)1 << 31 || p.N >= (int64_t)1 << 31 || p.K >= (int64_t)1 << 31)
    return PFLU_OK;
  static bool attr_dev[64] = {};
  int attr_d = 0;
  CK(cudaGetDevice(&attr_d));
  bool& attr = attr_dev[attr_d & 63];
  if (!attr) {
    CK(cudaFuncSetAttribute(gemm_dmma_ws<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  CUtensorMap ta, tb;
  const cuuint32_t es[2] = {1, 1};
  const cuuint64_t da[2] = {(cuuint64_t)p.K, (cuuint64_t)p.M}, sa[1] = {(cuuint64_t)p.lda * 8};
  const cuuint32_t ba[2] = {8, (cuuint32_t)C::BM};
  CUresult r = enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p.a), da, sa, ba, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(PFLU_ERR_CUDA, "cuTensorMapEncodeTiled(A) failed: %d", (int)r);
  const cuuint64_t db[2] = {(cuuint64_t)p.N, (cuuint64_t)p.K}, sb[1] = {(cuuint64_t)p.ldb * 8};
  const cuuint32_t bb[2] = {8, (cuuint32_t)C::BK};
  r = enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p.b), db, sb, bb, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(PFLU_ERR_CUDA, "cuTensorMapEncodeTiled(B) failed: %d", (int)r);
  const int64_t tm = (p.M + C::BM - 1) / C::BM, tn = (p.N + C::BN - 1) / C::BN;
  if (tm * tn > INT_MAX) return set_err(PFLU_ERR_UNSUPPORTED, "gemm grid too large");
  TmaGemmArgs q;
  q.c = p.c; q.ldc = p.ldc; q.M = p.M; q.N = p.N; q.K = p.K;
  q.tiles_m = (int)tm; q.tiles_n = (int)tn;
  gemm_dmma_ws<C><<<(unsigned)(tm * tn), C::THREADS, C::SMEM, st>>>(ta, tb, q);
  *done = true;
  return PFLU_OK;
}
// PFLU_GEMM_WS: 1 = WS1 (default, the production trailing update), 0 / 2 / 3 = the other ring
// depths, -1 = the cp.async GEMM (gemm_dmma_t / PFLU_GEMM_VARIANT)
// persistent, SM-budgeted WS GEMM over an atomic tile queue (gemm_dmma_ws_pers): grid CTAs; views
// that TMA cannot describe fall back to the dynamic tile-per-CTA GEMM (correct, not partitioned)
template <class C>
static int launch_gemm_pers(const GemmArgs& p, const WsCtl& ctl, int grid, cudaStream_t st, bool* done) {
  *done = false;
  PfnEncodeTiled enc = tma_encoder();
  if (!enc) return PFLU_OK;
  if ((reinterpret_cast<uintptr_t>(p.a) & 15) || (reinterpret_cast<uintptr_t>(p.b) & 15) ||
      (reinterpret_cast<uintptr_t>(p.c) & 15) || (p.lda & 1) || (p.ldb & 1) || (p.ldc & 1) ||
      p.M >= (int64_t)1 << 31 || p.N >= (int64_t)1 << 31 || p.K >= (int64_t)1 << 31)
    return PFLU_OK;
  constexpr int SMEM = C::SMEM + 64;  // + the per-stage tile indices
  static bool attr_dev[64] = {};
  int attr_d = 0;
  CK(cudaGetDevice(&attr_d));
  if (!attr_dev[attr_d & 63]) {
    CK(cudaFuncSetAttribute(gemm_dmma_ws_pers<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    attr_dev[attr_d & 63] = true;
  }
  CUtensorMap ta, tb;
  const cuuint32_t es[2] = {1, 1};
  const cuuint64_t da[2] = {(cuuint64_t)p.K, (cuuint64_t)p.M}, sa[1] = {(cuuint64_t)p.lda * 8};
  const cuuint32_t ba[2] = {8, (cuuint32_t)C::BM};
  CUresult r = enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p.a), da, sa, ba, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(PFLU_ERR_CUDA, "cuTensorMapEncodeTiled(A) failed: %d", (int)r);
  const cuuint64_t db[2] = {(cuuint64_t)p.N, (cuuint64_t)p.K}, sb[1] = {(cuuint64_t)p.ldb * 8};
  const cuuint32_t bb[2] = {8, (cuuint32_t)C::BK};
  r = enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p.b), db, sb, bb, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(PFLU_ERR_CUDA, "cuTensorMapEncodeTiled(B) failed: %d", (int)r);
  const int64_t tm = (p.M + C::BM - 1) / C::BM, tn = (p.N + C::BN - 1) / C::BN;
  if (tm * tn > INT_MAX) return set_err(PFLU_ERR_UNSUPPORTED, "gemm grid too large");
  TmaGemmArgs q;
  q.c = p.c; q.ldc = p.ldc; q.M = p.M; q.N = p.N; q.K = p.K;
  q.tiles_m = (int)tm; q.tiles_n = (int)tn;
  gemm_dmma_ws_pers<C><<<(unsigned)std::max(1, grid), C::THREADS, SMEM, st>>>(ta, tb, q, ctl);
  CK(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
  *done = true;
  return PFLU_OK;
}

static int g_gemm_ws = []() { const char* e = getenv("PFLU_GEMM_WS"); return e ? atoi(e) : 1; }();

static int launch_gemm(double* c, int64_t ldc, const double* a, int64_t lda, const double* b, int64_t ldb,
                       int64_t M, int64_t N, int64_t K, bool exact, cudaStream_t st, int pgrid = 0) {
  if (M <= 0 || N <= 0 || K <= 0) return PFLU_OK;
  GemmArgs p;
  p.c = c; p.a = a; p.b = b;
  p.ldc = ldc; p.lda = lda; p.ldb = ldb;
  p.M = M; p.N = N; p.K = K;
  const bool v2 = aligned16(c) && aligned16(a) && aligned16(b) && (ldc % 2 == 0) && (lda % 2 == 0) &&
                  (ldb % 2 == 0);
  if (exact) {
    int64_t tm = (M + GM_BM - 1) / GM_BM, tn = (N + GM_BN - 1) / GM_BN;
    if (tm * tn > INT_MAX) return set_err(PFLU_ERR_UNSUPPORTED, "gemm grid too large");
    p.tiles_m = (int)tm;
    p.tiles_n = (int)tn;
    dim3 grid((unsigned)(tm * tn));
    if (v2) gemm_exact_kernel<2><<<grid, GM_THREADS, GM_SMEM, st>>>(p);
    else gemm_exact_kernel<1><<<grid, GM_THREADS, GM_SMEM, st>>>(p);
  } else {
    bool done = false;
    switch (g_gemm_ws) {
      case 0: CKR(launch_gemm_ws<WS0>(p, st, &done)); break;
      case 1: CKR(launch_gemm_ws<WS1>(p, st, &done)); break;
      case 2: CKR(launch_gemm_ws<WS2>(p, st, &done)); break;
      case 3: CKR(launch_gemm_ws<WS3>(p, st, &done)); break;
      default: break;
    }
    if (!done && g_gemm_tma) CKR(launch_gemm_tma<GV6>(p, st, &done));
    if (!done) switch (g_gemm_variant) {
      case 1: CKR(launch_gemm_t<GV1>(p, v2, st)); break;
      case 2: CKR(launch_gemm_t<GV2>(p, v2, st)); break;
      case 3: CKR(launch_gemm_t<GV3>(p, v2, st)); break;
      case 4: CKR(launch_gemm_t<GV4>(p, v2, st)); break;
      case 5: CKR(launch_gemm_t<GV5>(p, v2, st)); break;
      case 6: CKR(launch_gemm_t<GV6>(p, v2, st)); break;
      case 7: CKR(launch_gemm_t<GV7>(p, v2, st)); break;
      case 10: CKR(launch_gemm_p<GV0>(*g_dc, p, v2, 0, st)); break;
      case 11: CKR((launch_gemm_p<GV0, true>(*g_dc, p, v2, 0, st))); break;
      case 13: CKR(launch_gemm_p<GV3>(*g_dc, p, v2, 0, st)); break;
      case 16: CKR(launch_gemm_p<GV6>(*g_dc, p, v2, 0, st)); break;
      case 8: CKR(launch_gemm_t<GV8>(p, v2, st)); break;
      case 9: CKR(launch_gemm_t<GV9>(p, v2, st)); break;
      case 40: CKR(launch_gemm_t<GV0>(p, v2, st)); break;
      case 17: CKR(launch_gemm_p<GV7>(*g_dc, p, v2, 0, st)); break;
      case 20: CKR(launch_gemm_p<GV0>(*g_dc, p, v2, g_dc->sms, st)); break;
      case 21: CKR(launch_gemm_p<GV3>(*g_dc, p, v2, g_dc->sms, st)); break;
      case 41:  // round-1 depth-0 choice (persistent GV0)
        if (pgrid != 0) CKR(launch_gemm_p<GV0>(*g_dc, p, v2, pgrid > 0 ? pgrid : 0, st));
        else CKR(launch_gemm_t<GV0>(p, v2, st));
        break;
      case 0:
      default: CKR(launch_gemm_t<GV6>(p, v2, st)); break;
    }
  }
  CK(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return PFLU_OK;
}

static int launch_trsm(const double* L, int64_t ldl, int np, double* X, int64_t ldx, int64_t ncols,
                       cudaStream_t st) {
  if (np <= 1 || ncols <= 0) return PFLU_OK;
  if (np > PLAN_MAX) return set_err(PFLU_ERR_UNSUPPORTED, "trsm block %d > %d", np, PLAN_MAX);
  if (np <= 256) {
    size_t smem = (size_t)(np * 32 + std::max(np, 32) * 32) * 8;
    trsm_kernel<32><<<(unsigned)((ncols + 31) / 32), 256, smem, st>>>(L, ldl, X, ldx, np, ncols);
  } else if (np <= 512) {
    size_t smem = (size_t)(np * 16 + std::max(np, 16) * 16) * 8;
    trsm_kernel<16><<<(unsigned)((ncols + 15) / 16), 256, smem, st>>>(L, ldl, X, ldx, np, ncols);
  } else {
    size_t smem = (size_t)(np * 8 + std::max(np, 8) * 8) * 8;
    trsm_kernel<8><<<(unsigned)((ncols + 7) / 8), 256, smem, st>>>(L, ldl, X, ldx, np, ncols);
  }
  CK(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return PFLU_OK;
}

static int launch_plan(const int64_t* piv, int64_t d, int np, int64_t* plan, cudaStream_t st) {
  if (np > PLAN_MAX) return set_err(PFLU_ERR_UNSUPPORTED, "pivot block %d > %d", np, PLAN_MAX);
  pivot_plan_kernel<<<1, 256, 0, st>>>(piv, d, np, plan);
  CK(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return PFLU_OK;
}

static int launch_diag_inv(const double* L, int64_t ldl, int np, double* inv, cudaStream_t st) {
  diag_inv_kernel<<<2, 128, 0, st>>>(L, ldl, np, inv);
  CK(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return PFLU_OK;
}

// laswp by plan (+ optional trsm) on storage columns [c0, c1); with `inv` (the inverted diagonal
// blocks of L, np <= 256) the solve runs on the tensor cores (fast mode)
static int launch_swap(double* a, int64_t lda, int64_t d, int np, const int64_t* plan, int64_t c0, int64_t c1,
                       const double* L, int64_t ldl, bool do_trsm, cudaStream_t st, const double* inv = nullptr) {
  if (c1 <= c0 || np <= 0) return PFLU_OK;
  const int t = do_trsm ? 1 : 0;
  if (do_trsm && inv && np <= 256 && g_swap_bn == 16) {
    swap_trsm_dmma_kernel<256, 16><<<(unsigned)((c1 - c0 + 15) / 16), 256, SdCfg<256, 16>::SMEM, st>>>(
        a, lda, d, np, plan, c0, c1, L, ldl, inv);
  } else if (do_trsm && inv && np <= 256) {
    swap_trsm_dmma_kernel<256, 32><<<(unsigned)((c1 - c0 + 31) / 32), 256, SdCfg<256, 32>::SMEM, st>>>(
        a, lda, d, np, plan, c0, c1, L, ldl, inv);
  } else if (do_trsm && inv && np <= 512) {
    swap_trsm_dmma_kernel<512, 16><<<(unsigned)((c1 - c0 + 15) / 16), 256, SdCfg<512, 16>::SMEM, st>>>(
        a, lda, d, np, plan, c0, c1, L, ldl, inv);
  } else if (!do_trsm && np <= 256 && g_lswap_tw == 8) {
    size_t smem = (size_t)(np * 8 + std::max(np * 8, 1024)) * 8;
    swap_trsm_kernel<8><<<(unsigned)((c1 - c0 + 7) / 8), 256, smem, st>>>(a, lda, d, np, plan, c0, c1, L, ldl, t);
  } else if (!do_trsm && np <= 256 && g_lswap_tw == 16) {
    // pure row permutation (the deferred left swaps, concurrent with the trailing GEMM): 16-column
    // strips (one 128-byte line per row), 64 KB of staging -> 3 CTAs per SM, twice the CTAs
    size_t smem = (size_t)(np * 16 + std::max(np * 16, 1024)) * 8;
    swap_trsm_kernel<16><<<(unsigned)((c1 - c0 + 15) / 16), 256, smem, st>>>(a, lda, d, np, plan, c0, c1, L, ldl, t);
  } else if (np <= 256) {
    size_t smem = (size_t)(np * 32 + std::max(np * 32, 1024)) * 8;
    swap_trsm_kernel<32><<<(unsigned)((c1 - c0 + 31) / 32), 256, smem, st>>>(a, lda, d, np, plan, c0, c1, L, ldl, t);
  } else if (np <= 512) {
    size_t smem = (size_t)(np * 16 + std::max(np * 16, 1024)) * 8;
    swap_trsm_kernel<16><<<(unsigned)((c1 - c0 + 15) / 16), 256, smem, st>>>(a, lda, d, np, plan, c0, c1, L, ldl, t);
  } else {
    size_t smem = (size_t)(np * 8 + std::max(np * 8, 1024)) * 8;
    swap_trsm_kernel<8><<<(unsigned)((c1 - c0 + 7) / 8), 256, smem, st>>>(a, lda, d, np, plan, c0, c1, L, ldl, t);
  }
  CK(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return PFLU_OK;
}

static int pf_occupancy(int W, size_t smem, int* occ) {
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, pf_fn(W, false), PF_THREADS, smem));
  return PFLU_OK;
}

static size_t pf_smem_bytes(int W, int64_t R, int w, bool cl = false) {
  if (W == 8) return PanelSmem<8>::bytes(R, w, cl);
  if (W == 16) return PanelSmem<16>::bytes(R, w, cl);
  return PanelSmem<32>::bytes(R, w, cl);
}
static int64_t pf_swap_doubles(int W, int w) {
  return W == 8 ? PanelSmem<8>::swap_doubles(w) : W == 16 ? PanelSmem<16>::swap_doubles(w) : PanelSmem<32>::swap_doubles(w);
}

// can a cluster of S panel CTAs (W, full shared memory) be resident?  cached per (W, S)
static int pf_cluster_ok(DevCtx& c, int W, int S, bool* ok) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  static int cache[3][PF_CL_MAX + 1];
  static bool init = false;
  if (!init) {
    for (auto& r : cache)
      for (int& v : r) v = -1;
    init = true;
  }
  const int wi = W == 8 ? 0 : W == 16 ? 1 : 2;
  if (cache[wi][S] < 0) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = S;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(S);
    cfg.blockDim = dim3(PF_THREADS);
    cfg.dynamicSmemBytes = c.smem_optin - 2048;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, pf_fn(W, true), &cfg);
    if (e != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    cache[wi][S] = n;
  }
  *ok = cache[wi][S] > 0;
  return PFLU_OK;
}

// Persistent panel factorization: rows [r0, m) of storage columns [c0, c0 + w).
static int panel_leaf(DevCtx& c, double* a, int64_t lda, int64_t m, int64_t r0, int64_t c0, int64_t w,
                        int64_t* piv, unsigned long long* info, const pflu_options& opt, cudaStream_t st) {
  const int64_t rows = m - r0;
  if (rows <= 0 || w <= 0) return PFLU_OK;
  const size_t smax = c.smem_optin - 2048;
  int Wpref = opt.leaf_width > 0 ? opt.leaf_width : g_leaf > 0 ? g_leaf : (w > 16 ? 32 : (w > 8 ? 16 : 8));
  const int Ws[3] = {32, 16, 8};
  PanelArgs p;
  p.a = a; p.lda = lda; p.m = m; p.r0 = r0; p.col0 = c0; p.w = (int)w;
  p.piv = piv; p.info = info; p.ll = c.ll; p.epoch = c.epoch; p.exact = opt.exact;
  p.prof = g_prof;
  p.resync = g_resync;
  p.swcap = 0;
  p.sm_mask = c.rec_mask;
  c.rec_mask = nullptr;  // only the first persistent launch of a (split) panel records its SMs
  // several 16-CTA clusters (panel_kernel 4): v2 exchange inside each cluster, one LL round between them
  if (opt.panel_kernel == 4 && g_pf_v2 != 0 && rows >= g_mc_minrows) {
    // panel_ctas > 0 caps the CTAs, i.e. the clusters (at least two)
    const int cl_cap = opt.panel_ctas > 0 ? std::max(2, std::min(g_mc_maxcl, opt.panel_ctas / PF_CL_MAX)) : g_mc_maxcl;
    for (int wi = 0; wi < 3; ++wi) {
      const int W = Ws[wi];
      if (W > Wpref) continue;
      int NC = (int)std::min<int64_t>(cl_cap, std::max<int64_t>(2, (rows + g_mc_rows - 1) / g_mc_rows));
      const int64_t R = (rows + (int64_t)NC * PF_CL_MAX - 1) / ((int64_t)NC * PF_CL_MAX);
      const size_t smem = pf_smem_bytes(W, R, (int)w, true);
      if (smem > smax) continue;
      NC = (int)((rows + R * PF_CL_MAX - 1) / (R * PF_CL_MAX));  // clusters that own rows
      if (NC < 2) break;
      p.R = R;
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = PF_CL_MAX;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative;  // every cluster resident: they wait for one another
      at[1].val.cooperative = 1;
      cfg.gridDim = dim3(NC * PF_CL_MAX);
      cfg.blockDim = dim3(PF_THREADS);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      void* args[] = {&p};
      // The clusters wait for one another: launch only what the device can hold at once (16-CTA clusters
      // need 16 free SMs inside one GPC) and only cooperatively; otherwise the grid kernel below runs.
      int max_cl = 0;
      if (cudaOccupancyMaxActiveClusters(&max_cl, pf_fn(W, true, opt.exact != 0, true, true), &cfg) != cudaSuccess) {
        cudaGetLastError();
        max_cl = 0;
      }
      if (max_cl < NC) break;
      if (cudaLaunchKernelExC(&cfg, pf_fn(W, true, opt.exact != 0, true, true), args) != cudaSuccess) {
        cudaGetLastError();
        break;
      }
      g_launches.fetch_add(1, std::memory_order_relaxed);
      return PFLU_OK;
    }
  }
  // one thread-block cluster (DSMEM exchange) when the rows fit its CTAs' shared memory
  const bool want_cl = opt.panel_kernel == 2 || (opt.panel_kernel == 0 && g_cluster > 0 && rows <= g_cl_rows);
  if (want_cl) {
    const int Smax = opt.panel_ctas > 0 ? std::min(opt.panel_ctas, PF_CL_MAX)
                                        : std::max(1, std::min(g_cluster > 0 ? g_cluster : PF_CL_MAX, PF_CL_MAX));
    for (int wi = 0; wi < 3; ++wi) {
      const int W = Ws[wi];
      if (W > Wpref) continue;
      const int S0 = (int)std::min<int64_t>(Smax, std::max<int64_t>(1, (rows + g_cl_minrows - 1) / g_cl_minrows));
      const int64_t R = (rows + S0 - 1) / S0;
      const int S = (int)((rows + R - 1) / R);
      size_t smem = pf_smem_bytes(W, R, (int)w, true);
      if (smem > smax) continue;
      // dedicated row-swap staging from the shared memory left over (small panels)
      const int64_t swcap = std::min<int64_t>(pf_swap_doubles(W, (int)w), (int64_t)(smax - smem) / 8);
      p.swcap = swcap > 0 ? (int)swcap : 0;
      smem += (size_t)p.swcap * 8;
      bool ok = false;
      CKR(pf_cluster_ok(c, W, S, &ok));
      if (!ok) continue;
      p.R = R;
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = S;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(S);
      cfg.blockDim = dim3(PF_THREADS);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      void* args[] = {&p};
      // peers: the v2 leaf (dedicated exchange warp, per-warp candidates); a one-CTA cluster has no exchange
      CK(cudaLaunchKernelExC(&cfg, pf_fn(W, true, opt.exact != 0, g_pf_v2 != 0 && S > 1), args));
      g_launches.fetch_add(1, std::memory_order_relaxed);
      return PFLU_OK;
    }
    if (opt.panel_kernel == 2)
      return set_err(PFLU_ERR_UNSUPPORTED, "panel of %lld rows x %lld does not fit one thread-block cluster",
                     (long long)rows, (long long)w);
  }
  for (int wi = 0; wi < 3; ++wi) {
    const int W = Ws[wi];
    if (W > Wpref) continue;
    // tall panels: 64 CTAs (measured: 32768 x 256 1.65 -> 1.50 ms, 16384 x 256 1.33 -> 1.21 ms)
    const int cap = rows >= 16384 ? std::max(g_pf_cap, 64) : g_pf_cap;
    int S = opt.panel_ctas > 0 ? opt.panel_ctas : (int)std::min<int64_t>(cap, (rows + 255) / 256);
    S = std::max(1, std::min(S, PF_MAX_CTAS));
    for (; S <= PF_MAX_CTAS; ++S) {
      const int64_t R = (rows + S - 1) / S;
      const size_t smem = pf_smem_bytes(W, R, (int)w);
      if (smem > smax) continue;
      int occ = 0;
      CKR(pf_occupancy(W, smem, &occ));
      if ((int64_t)occ * c.sms < S) break;
      int S_eff = (int)((rows + R - 1) / R);
      p.R = R;
      void* args[] = {&p};
      CK(cudaLaunchCooperativeKernel(pf_fn(W, false, opt.exact != 0), dim3(S_eff), dim3(PF_THREADS), args, smem, st));
      g_launches.fetch_add(1, std::memory_order_relaxed);
      return PFLU_OK;
    }
  }
  return set_err(PFLU_ERR_UNSUPPORTED, "panel of %lld rows x %lld does not fit the persistent panel kernel",
                 (long long)rows, (long long)w);
}

// Recursive panel (panel_kernel 3; Toledo's recursive LU restricted to the panel's columns):
//   left half recursively -> its swaps + U12 := L11^-1 A12 on the right half (swap+TRSM kernel) ->
//   A22 -= L21 U12 over the full panel height (DMMA GEMM on every free SM) -> right half
//   recursively -> its swaps applied back to the left half's columns.
// Leaves of <= g_rec_leaf columns run on the persistent panel kernel.  Every element still receives
// its updates in ascending pivot order (multiply, then subtract in exact mode), so exact mode stays
// bitwise equal to the unblocked getf2 of the reference (_jit.py:154-187), like the outer blocking.
static int panel_rec(DevCtx& c, double* a, int64_t lda, int64_t m, int64_t r0, int64_t c0, int64_t w,
                     int64_t* piv, unsigned long long* info, const pflu_options& opt, cudaStream_t st,
                     int leaf, int leafk) {
  const int64_t rows = m - r0;
  if (rows <= 0 || w <= 0) return PFLU_OK;
  if (w <= leaf) {
    pflu_options lo = opt;
    lo.panel_kernel = leafk;
    return panel_leaf(c, a, lda, m, r0, c0, w, piv, info, lo, st);
  }
  // split at a multiple of the leaf width near the middle
  int64_t h = ((w / 2 + leaf - 1) / leaf) * leaf;
  if (h >= w) h = w - leaf;
  CKR(panel_rec(c, a, lda, m, r0, c0, h, piv, info, opt, st, leaf, leafk));
  const int np = (int)std::min<int64_t>(h, rows);
  const bool exact = opt.exact != 0;
  CKR(launch_plan(piv, r0, np, c.rplan, st));
  const double* l11 = a + r0 * lda + c0;
  const bool dinv = !exact && g_trsm_dmma && np <= 512;
  if (dinv) CKR(launch_diag_inv(l11, lda, np, c.rinv, st));
  CKR(launch_swap(a, lda, r0, np, c.rplan, c0 + h, c0 + w, l11, lda, true, st, dinv ? c.rinv : nullptr));
  if (rows <= np) return PFLU_OK;
  CKR(launch_gemm(a + (r0 + np) * lda + c0 + h, lda, a + (r0 + np) * lda + c0, lda, a + r0 * lda + c0 + h, lda,
                  rows - np, w - h, np, exact, st));
  CKR(panel_rec(c, a, lda, m, r0 + np, c0 + h, w - h, piv, info, opt, st, leaf, leafk));
  const int np2 = (int)std::min<int64_t>(w - h, rows - np);
  CKR(launch_plan(piv, r0 + np, np2, c.rplan, st));
  return launch_swap(a, lda, r0 + np, np2, c.rplan, c0, c0 + h, nullptr, lda, false, st);
}

static int panel_factor(DevCtx& c, double* a, int64_t lda, int64_t m, int64_t r0, int64_t c0, int64_t w,
                        int64_t* piv, unsigned long long* info, const pflu_options& opt, cudaStream_t st) {
  if (opt.panel_kernel == 3)
    return panel_rec(c, a, lda, m, r0, c0, w, piv, info, opt, st, std::max(8, g_rec_leaf), g_rec_leafk);
  // Automatic top-level split (round 2): a panel of >= 2 x 128 columns and >= 4096 rows is factored as
  // two 128-column halves on the persistent kernel the caller chose (automatic / grid / cluster), with
  // the right half's swap + U12 solve + rank-128 update between them on the DMMA kernels that own every
  // SM -- half of the in-panel update leaves the panel kernel's 16 (or 64) SMs.  Measured alone on the
  // GPU (profiles/r06_panel_sweep.log): 8192 x 256 0.840 -> 0.759 ms, 16384 x 256 1.456 -> 1.106,
  // 32768 x 256 (grid leaves) 1.446 -> 1.299.  Exact mode stays bitwise (same per-element update order).
  // (Every schedule splits alike -- also the SM-partitioned ones -- so that all of them stay bitwise equal.)
  if (g_auto_rec_leaf > 0 && w >= 2 * g_auto_rec_leaf && m - r0 >= g_auto_rec_minrows &&
      (opt.panel_ctas == 0 || opt.panel_kernel == 4) && opt.leaf_width == 0)
    return panel_rec(c, a, lda, m, r0, c0, w, piv, info, opt, st, g_auto_rec_leaf, opt.panel_kernel);
  return panel_leaf(c, a, lda, m, r0, c0, w, piv, info, opt, st);
}

// ------------------------------------------------------------------------------------------
// the blocked factorization

struct Step {
  int64_t col0, bw;
};

// Called when rows [r0, r1) of the matrix are final (every later step only touches rows below),
// after the work on stream `after`; lets pflu_getrf stream results to the host during the run.
using RowSink = std::function<int(int64_t r0, int64_t r1, cudaStream_t after)>;
// Host source of the matrix for pflu_getrf (look-ahead 1): the H2D is issued per trailing-update
// column chunk on the caller's stream, and each chunk's work waits only for its own columns, so
// the transfer of later columns overlaps the first steps on earlier ones.
struct HostIn {
  const double* a;
  int64_t lda;
  int chunks;
};
static int g_h2d_chunks = []() { const char* e = getenv("PFLU_H2D_CHUNKS"); return e ? atoi(e) : 6; }();  // e2e: 4 -> 819.5, 5 -> 815.5, 6 -> 812.9, 8 -> 891 ms

static int getrf_async(DevCtx& c, double* a, int64_t m, int64_t n, int64_t lda, int64_t b, int lookahead,
                       int64_t* piv, unsigned long long* info, cudaStream_t user, const pflu_options& opt,
                       Tracer& tr, const RowSink* sink = nullptr, const HostIn* hin = nullptr) {
  std::vector<Step> grid;
  for (int64_t col0 = 0; col0 < n; col0 += b) grid.push_back({col0, std::min(b, n - col0)});
  const int count = (int)grid.size();
  const bool exact = opt.exact != 0;
  CK(cudaMemsetAsync(info, 0xff, sizeof(unsigned long long), user));
  CKR(tr.start(user));
  // per-step pivot plans (no reuse hazards between concurrently running steps)
  const size_t plan_words = 1 + 3 * (size_t)std::max<int64_t>(1, std::min(b, n));
  if (c.plans_cap < plan_words * count) {
    if (c.plans) CK(cudaFree(c.plans));
    c.plans_cap = plan_words * count;
    CK(cudaMalloc(&c.plans, sizeof(int64_t) * c.plans_cap));
  }
  auto plan_of = [&](int k) { return c.plans + plan_words * k; };
  // fast mode: inverted 32x32 diagonal blocks of each step's L11 for the DMMA solve
  const bool use_dinv = !exact && g_trsm_dmma && std::min(b, n) <= 512;
  const size_t inv_words = (size_t)1024 * ((std::min(b, n) + 31) / 32);  // one 32x32 block per 32 rows
  if (use_dinv && c.dinv_cap < inv_words * count) {
    if (c.dinv) CK(cudaFree(c.dinv));
    c.dinv_cap = inv_words * count;
    CK(cudaMalloc(&c.dinv, sizeof(double) * c.dinv_cap));
  }
  auto inv_of = [&](int k) { return c.dinv + inv_words * k; };
  // SM-partitioned look-ahead (pflu_options.malleable 1 = LA, 2 = LA_MB; DMMA mode, look-ahead 1):
  // TU_R(k)'s GEMM is a persistent kernel over tile queue k that leaves the panel's SMs alone
  const int sched = (lookahead == 1 && !exact && !g_tur_split && !g_emu_ranks) ? std::max(0, std::min(2, opt.malleable)) : 0;
  if (sched) {
    if (!c.sm_mask) CK(cudaMalloc(&c.sm_mask, 8 * sizeof(unsigned)));
    if (c.tile_ctr_cap < (size_t)count) {
      if (c.tile_ctr) CK(cudaFree(c.tile_ctr));
      c.tile_ctr = nullptr;
      c.tile_ctr_cap = 0;
      CK(cudaMalloc(&c.tile_ctr, sizeof(int) * count));
      c.tile_ctr_cap = count;
    }
    CK(cudaMemsetAsync(c.sm_mask, 0, 8 * sizeof(unsigned), user));
    CK(cudaMemsetAsync(c.tile_ctr, 0, sizeof(int) * count, user));
    while (c.swev.size() < (size_t)count) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c.swev.push_back(e);
    }
  }
  // the trailing GEMM of TU_R(k) on [lo, hi) as a persistent kernel (main grid or the join grid)
  auto tur_gemm_pers = [&](int k, int64_t lo, int64_t hi, bool joiner, cudaStream_t st, bool* done) -> int {
    *done = false;
    const Step s = grid[k];
    const int64_t below = s.col0 + s.bw;
    if (hi <= lo || below >= m) return PFLU_OK;
    GemmArgs gp;
    gp.c = a + below * lda + lo; gp.a = a + below * lda + s.col0; gp.b = a + s.col0 * lda + lo;
    gp.ldc = lda; gp.lda = lda; gp.ldb = lda;
    gp.M = m - below; gp.N = hi - lo; gp.K = s.bw;
    const WsCtl ctl{c.tile_ctr + k, c.sm_mask, joiner ? 1 : 0};
    return launch_gemm_pers<WS1>(gp, ctl, joiner ? 2 * PF_CL_MAX : 2 * c.sms, st, done);
  };
  auto update_cols = [&](int k, int64_t lo, int64_t hi, cudaStream_t st, int label) -> int {
    // TU of step k on storage columns [lo, hi): laswp + trsm (fused), then the DMMA update
    if (hi <= lo) return PFLU_OK;
    const Step s = grid[k];
    const int np = (int)std::min(s.bw, m - s.col0);
    int t_tu = -1, t_g = -1;
    CKR(tr.begin(label, k, st, &t_tu));
    CKR(launch_swap(a, lda, s.col0, np, plan_of(k), lo, hi, a + s.col0 * lda + s.col0, lda, true, st,
                    use_dinv ? inv_of(k) : nullptr));
    const int64_t below = s.col0 + s.bw;
    if (below < m) {
      if (label != PFLU_TRACE_TU_L)
        CKR(tr.begin(PFLU_TRACE_GEMM, k, st, &t_g, 2.0 * (double)(m - below) * (double)(hi - lo) * (double)s.bw));
      const int pg = label == PFLU_TRACE_TU ? -1 : (label == PFLU_TRACE_TU_R ? g_tur_grid : 0);
      bool done = false;
      if (sched && label == PFLU_TRACE_TU_R) {
        CK(cudaEventRecord(c.swev[k], st));  // the join grid may take tiles once U12 is solved
        CKR(tur_gemm_pers(k, lo, hi, false, st, &done));
      }
      if (!done)
        CKR(launch_gemm(a + below * lda + lo, lda, a + below * lda + s.col0, lda, a + s.col0 * lda + lo, lda,
                        m - below, hi - lo, s.bw, exact, st, pg));
      CKR(tr.end(t_g, st));
    }
    return tr.end(t_tu, st);
  };
  auto left_swaps = [&](int k, cudaStream_t st) -> int {
    const Step s = grid[k];
    if (s.col0 == 0) return PFLU_OK;
    const int np = (int)std::min(s.bw, m - s.col0);
    const int64_t hi = g_emu_ranks > 1 ? std::min<int64_t>(s.col0, (s.col0 / g_emu_ranks + b - 1) / b * b) : s.col0;
    return launch_swap(a, lda, s.col0, np, plan_of(k), 0, hi, nullptr, lda, false, st);
  };
  // Depth 0 runs each panel alone on the critical path: tall panels take the cooperative-grid kernel
  // (more SMs, lower latency).  Depth 1 keeps the 16-SM cluster kernel, which leaves the other SMs to
  // the concurrent trailing update.
  auto pf = [&](int k, cudaStream_t st) -> int {
    const Step s = grid[k];
    int t_pf = -1;
    CKR(tr.begin(PFLU_TRACE_PF, k, st, &t_pf));
    pflu_options popt = opt;
    if (lookahead == 0 && popt.panel_kernel == 0 && m - s.col0 > g_grid_rows) popt.panel_kernel = g_tall_kernel;
    // = dist.py: the owner's tall panels on the grid kernel from 8 ranks up (chain-bound there)
    if (g_emu_ranks >= g_emu_grid_ranks && popt.panel_kernel == 0 && m - s.col0 > g_grid_rows) {
      popt.panel_kernel = g_tall_kernel;
      if (g_tall_kernel == 4 && popt.panel_ctas == 0 && g_mc_adapt)
        popt.panel_ctas = tall_panel_ctas(m - s.col0, (n - s.col0 - s.bw) / g_emu_ranks, s.bw);
    }
    // depth 1, single rank: panels taller than PFLU_LA_TALL_ROWS leave the 16-SM cluster for the tall-panel kernel
    if (lookahead != 0 && popt.panel_kernel == 0 && m - s.col0 > g_la_tall_rows) popt.panel_kernel = g_tall_kernel;
    if (g_pf_force >= 0 && opt.panel_kernel == 0) popt.panel_kernel = g_pf_force;
    if (sched && k == 0) c.rec_mask = c.sm_mask;  // PF(0) runs alone: its SMs become the panel's partition
    const int prc = panel_factor(c, a, lda, m, s.col0, s.col0, s.bw, piv, info, popt, st);
    c.rec_mask = nullptr;
    CKR(prc);
    const int np = (int)std::min(s.bw, m - s.col0);
    CKR(launch_plan(piv, s.col0, np, plan_of(k), st));
    if (use_dinv) CKR(launch_diag_inv(a + s.col0 * lda + s.col0, lda, np, inv_of(k), st));
    return tr.end(t_pf, st);
  };

  if (lookahead == 0) {
    // dmf_mtb order (factor.py:396-411): PF(k), left swaps, TU on [col0+bw, n)
    for (int k = 0; k < count; ++k) {
      CKR(pf(k, user));
      CKR(left_swaps(k, user));
      CKR(update_cols(k, grid[k].col0 + grid[k].bw, n, user, PFLU_TRACE_TU));
      if (sink && k + 1 < count) CKR((*sink)(grid[k].col0, grid[k].col0 + grid[k].bw, user));
    }
    return PFLU_OK;
  }
  // lookahead 1, split-overlap schedule (PFLU_TUR_SPLIT=1, device buffers): the trailing columns of
  // every step are cut into a left part [lo_r, q) and a right part [q, n) at a boundary q taken from
  // the fixed sequence n/2, 3n/4, 7n/8, ... (the first one right of lo_r), so every part is contained
  // in one part of the previous step.  All GEMMs run in order on ONE stream (no concurrent GEMMs),
  // all swap+TRSMs on another: the swap+TRSM of step k's left part runs while GEMM(k-1)'s right
  // part computes, and step k's right part while GEMM(k)'s left part computes.
  if (g_tur_split && !hin && !sink) {
    cudaStream_t sG = c.sC[0], sS = c.sC[1];
    std::vector<int64_t> qs;  // boundary sequence (block aligned), ascending
    for (int64_t lo = 0, q; ; lo = q) {
      q = std::min<int64_t>(n, ((lo + (n - lo) / 2) + b - 1) / b * b);
      if (q <= lo || q >= n) break;
      qs.push_back(q);
    }
    auto bound_of = [&](int64_t lo_r) -> int64_t {  // right end of the left part
      for (int64_t q : qs)
        if (q > lo_r) return q;
      return n;
    };
    // events: [k][0] PF done, [k][1] TU_L done, [k][2..3] swap parts, [k][4..5] GEMM parts
    const size_t ne = 6;
    CKR(ctx_events(c, 2 + (size_t)count * ne));
    auto evk = [&](int k, int i) { return c.ev[2 + (size_t)k * ne + i]; };
    std::vector<int64_t> pb((size_t)count * 3);  // per step: lo_r, q, hi
    for (int k = 0; k < count; ++k) {
      const int64_t lo_r = (k + 1 < count) ? grid[k + 1].col0 + grid[k + 1].bw : n;
      int64_t hi_r = n;
      if (g_emu_ranks > 1) hi_r = std::min<int64_t>(n, lo_r + ((n - lo_r + g_emu_ranks - 1) / g_emu_ranks + b - 1) / b * b);
      pb[3 * k] = lo_r;
      pb[3 * k + 1] = std::min(bound_of(lo_r), hi_r);
      pb[3 * k + 2] = hi_r;
    }
    // which part of step k contains column col (0 left, 1 right, -1 none)
    auto part_of = [&](int k, int64_t col) -> int {
      if (col < pb[3 * k] || col >= pb[3 * k + 2]) return -1;
      return col < pb[3 * k + 1] ? 0 : 1;
    };
    cudaEvent_t ev_start = c.ev[0];
    CK(cudaEventRecord(ev_start, user));
    for (cudaStream_t st : {c.sP, c.sL, sG, sS}) CK(cudaStreamWaitEvent(st, ev_start, 0));
    CKR(pf(0, c.sP));
    CK(cudaEventRecord(evk(0, 0), c.sP));
    for (int k = 0; k < count; ++k) {
      const Step sk = grid[k];
      const int np = (int)std::min(sk.bw, m - sk.col0);
      const int64_t below = sk.col0 + sk.bw;
      for (int part = 0; part < 2; ++part) {
        const int64_t lo = part == 0 ? pb[3 * k] : pb[3 * k + 1], hi = part == 0 ? pb[3 * k + 1] : pb[3 * k + 2];
        if (hi > lo) {
          CK(cudaStreamWaitEvent(sS, evk(k, 0), 0));
          if (k > 0)  // the GEMM(k-1) part(s) that wrote these columns
            for (int pp = 0; pp < 2; ++pp) {
              const int64_t plo = pp == 0 ? pb[3 * (k - 1)] : pb[3 * (k - 1) + 1];
              const int64_t phi = pp == 0 ? pb[3 * (k - 1) + 1] : pb[3 * (k - 1) + 2];
              if (plo < hi && lo < phi) CK(cudaStreamWaitEvent(sS, evk(k - 1, 4 + pp), 0));
            }
          int t_s = -1;
          CKR(tr.begin(PFLU_TRACE_TU_R, k, sS, &t_s));
          CKR(launch_swap(a, lda, sk.col0, np, plan_of(k), lo, hi, a + sk.col0 * lda + sk.col0, lda, true, sS,
                          use_dinv ? inv_of(k) : nullptr));
          CKR(tr.end(t_s, sS));
        }
        CK(cudaEventRecord(evk(k, 2 + part), sS));
      }
      for (int part = 0; part < 2; ++part) {
        const int64_t lo = part == 0 ? pb[3 * k] : pb[3 * k + 1], hi = part == 0 ? pb[3 * k + 1] : pb[3 * k + 2];
        if (hi > lo && below < m) {
          CK(cudaStreamWaitEvent(sG, evk(k, 2 + part), 0));
          int t_g = -1;
          CKR(tr.begin(PFLU_TRACE_GEMM, k, sG, &t_g, 2.0 * (double)(m - below) * (double)(hi - lo) * (double)sk.bw));
          CKR(launch_gemm(a + below * lda + lo, lda, a + below * lda + sk.col0, lda, a + sk.col0 * lda + lo, lda,
                          m - below, hi - lo, sk.bw, exact, sG, g_tur_grid));
          CKR(tr.end(t_g, sG));
        }
        CK(cudaEventRecord(evk(k, 4 + part), sG));
      }
      if (k > 0) {  // left swaps(k): every reader of L21(k-1) finished
        CK(cudaStreamWaitEvent(c.sL, evk(k, 0), 0));
        CK(cudaStreamWaitEvent(c.sL, evk(k - 1, 4), 0));
        CK(cudaStreamWaitEvent(c.sL, evk(k - 1, 5), 0));
        CK(cudaStreamWaitEvent(c.sL, evk(k - 1, 1), 0));
        CKR(left_swaps(k, c.sL));
      }
      if (k + 1 < count) {
        if (k > 0) {  // block k+1 was last updated by GEMM(k-1)
          const int pp = part_of(k - 1, grid[k + 1].col0);
          if (pp >= 0) CK(cudaStreamWaitEvent(c.sP, evk(k - 1, 4 + pp), 0));
        }
        CKR(update_cols(k, grid[k + 1].col0, grid[k + 1].col0 + grid[k + 1].bw, c.sP, PFLU_TRACE_TU_L));
        CK(cudaEventRecord(evk(k, 1), c.sP));
        CKR(pf(k + 1, c.sP));
        CK(cudaEventRecord(evk(k + 1, 0), c.sP));
      } else {
        CK(cudaEventRecord(evk(k, 1), c.sP));
      }
    }
    CK(cudaEventRecord(c.ev[1], c.sP));
    CK(cudaStreamWaitEvent(user, c.ev[1], 0));
    for (cudaStream_t st : {sG, sS, c.sL}) {
      cudaEvent_t e = evk(count - 1, 2);  // reuse: recorded last on each stream in turn
      CK(cudaEventRecord(e, st));
      CK(cudaStreamWaitEvent(user, e, 0));
    }
    return PFLU_OK;
  }
  // lookahead 1 (dmf_la, factor.py:481-512) as a column-chunk dataflow.  The trailing columns are
  // split into NCH fixed, block-aligned chunks, each with its own stream that runs its part of every
  // step (laswp + trsm, then the GEMM) and depends only on the panel of that step -- a chunk never
  // waits for another chunk, so one chunk's swap/solve overlaps the others' GEMMs.
  //   sP (highest priority): TU_L(k) on block k+1 (after the chunk holding it finished step k-1),
  //                          PF(k+1), plan(k+1)
  //   sC[c]:                 TU_R(k) restricted to chunk c (after PF(k))
  //   sL:                    left swaps(k) on blocks < k (after every reader of L21(k-1) finished)
  // device buffers: 6 chunks up to n = 16384, where the panel chain still shows (C3 117.2 -> 115.1 ms,
  // C2 31.9 -> 31.6 ms: the panel stream only waits for the chunk that holds block k+1); one stream
  // above (C4 unchanged, its concurrent chunk GEMMs interfere); PFLU_CHUNKS overrides
  // r05 (WS GEMM) re-measure, profiles/r05_chunks_sweep.log: C4 1 chunk 723.2 ms, 2: 723.1, 3: 721.0,
  // 4: 719.8, 6: 720.0; C3 114.3 / 112.8 / 112.6 / 112.4 / 112.4 -> 6 up to 16384, 4 above
  // r06: 5 above 16384 -- same time as 4 (C4 705.9 vs 706.1 ms, C5 5472 vs 5473 ms) with the swap + U12-solve
  // time that no GEMM covers down from 6.9 to 4.2 ms (tools/exposed_swap.py; 6: 5.4 ms, 8: 4.7 ms but +4 ms)
  const int dflt = g_chunks_env > 0 ? g_chunks_env : (n <= 16384 ? 6 : 5);
  const int nch = sched ? 1 : std::max(1, std::min({hin ? std::max(dflt, hin->chunks) : dflt, MAX_CHUNKS, count}));
  std::vector<int> chunk_blk(nch + 1);
  for (int ch = 0; ch <= nch; ++ch) chunk_blk[ch] = (int)((int64_t)count * ch / nch);
  auto chunk_of_block = [&](int blk) {
    int ch = 0;
    while (ch + 1 < nch && chunk_blk[ch + 1] <= blk) ++ch;
    return ch;
  };
  // per step: PF, TU_L, first trailing block, then the chunks
  const size_t nev = 2 + (size_t)count * (nch + 3);
  CKR(ctx_events(c, nev + nch + 1));
  cudaEvent_t ev_start = c.ev[0];
  auto ev_pf = [&](int k) { return c.ev[2 + (size_t)k * (nch + 3)]; };
  auto ev_tul = [&](int k) { return c.ev[3 + (size_t)k * (nch + 3)]; };
  auto ev_first = [&](int k) { return c.ev[4 + (size_t)k * (nch + 3)]; };
  auto ev_ck = [&](int ch, int k) { return c.ev[5 + (size_t)k * (nch + 3) + ch]; };
  // PFLU_FIRST_BLOCK=1 (off: measured no gain): TU_R(k) updates block k+2 (the block TU_L(k+1) and PF(k+2)
  // need) as its own launch at the head of its chunk stream and TU_L(k+1) waits for that piece only.  The
  // stall it targets (8-rank model, early steps: 25 ms of PF -> TU_L gaps) is not a scheduling artefact: that
  // block's previous update sits inside the bulk of TU_R(k-1), and the chunk stream is in order, so while a
  // step's trailing update outlasts its panel the run is update-bound whatever the order (model 189.5 vs
  // 184.5 ms, C3 108.2 vs 102.8 ms with the extra launches).
  const bool first_blk = g_first_block != 0 && !sched;
  CK(cudaEventRecord(ev_start, user));
  CK(cudaStreamWaitEvent(c.sP, ev_start, 0));
  CK(cudaStreamWaitEvent(c.sL, ev_start, 0));
  for (int ch = 0; ch < nch; ++ch) CK(cudaStreamWaitEvent(c.sC[ch], ev_start, 0));
  if (hin) {  // per-chunk H2D on `user`, in column order
    // the first two block columns go first, on their own: PF(0), TU_L(0) and PF(1) touch only them,
    // so the panel chain starts while the rest of the first chunk is still in flight
    const int64_t head = std::min<int64_t>(n, 2 * b);
    CK(cudaMemcpy2DAsync(a, lda * 8, hin->a, hin->lda * 8, head * 8, m, cudaMemcpyHostToDevice, user));
    CK(cudaEventRecord(c.ev[nev + nch], user));
    CK(cudaStreamWaitEvent(c.sP, c.ev[nev + nch], 0));
    for (int ch = 0; ch < nch; ++ch) {
      const int64_t lo = std::max<int64_t>(head, (int64_t)chunk_blk[ch] * b);
      const int64_t hi = std::min<int64_t>(n, (int64_t)chunk_blk[ch + 1] * b);
      if (hi > lo)
        CK(cudaMemcpy2DAsync(a + lo, lda * 8, hin->a + lo, hin->lda * 8, (hi - lo) * 8, m, cudaMemcpyHostToDevice, user));
      cudaEvent_t e = c.ev[nev + ch];
      CK(cudaEventRecord(e, user));
      CK(cudaStreamWaitEvent(c.sC[ch], e, 0));
    }
  }
  CKR(pf(0, c.sP));
  CK(cudaEventRecord(ev_pf(0), c.sP));
  for (int k = 0; k < count; ++k) {
    const int64_t lo_r = (k + 1 < count) ? grid[k + 1].col0 + grid[k + 1].bw : n;
    int64_t hi_r = n;
    if (g_emu_ranks > 1) hi_r = std::min<int64_t>(n, lo_r + ((n - lo_r + g_emu_ranks - 1) / g_emu_ranks + b - 1) / b * b);
    for (int ch = 0; ch < nch; ++ch) {
      cudaStream_t st = c.sC[ch];
      const int64_t c_lo = std::max<int64_t>(lo_r, (int64_t)chunk_blk[ch] * b);
      const int64_t c_hi = std::min<int64_t>(hi_r, (int64_t)chunk_blk[ch + 1] * b);
      if (c_hi > c_lo) {
        CK(cudaStreamWaitEvent(st, ev_pf(k), 0));
        int64_t lo2 = c_lo;
        if (first_blk && c_lo == lo_r && k + 2 < count && c_hi > c_lo + grid[k + 2].bw) {
          lo2 = c_lo + grid[k + 2].bw;
          CKR(update_cols(k, c_lo, lo2, st, PFLU_TRACE_TU_R));
          CK(cudaEventRecord(ev_first(k), st));
        }
        CKR(update_cols(k, lo2, c_hi, st, PFLU_TRACE_TU_R));
        if (lo2 == c_lo && c_lo == lo_r) CK(cudaEventRecord(ev_first(k), st));
      }
      CK(cudaEventRecord(ev_ck(ch, k), st));
    }
    if (k > 0) {
      // left swaps(k) rewrite rows of L21(k-1): wait for every GEMM(k-1) (chunks + TU_L)
      CK(cudaStreamWaitEvent(c.sL, ev_pf(k), 0));
      for (int ch = 0; ch < nch; ++ch) CK(cudaStreamWaitEvent(c.sL, ev_ck(ch, k - 1), 0));
      CK(cudaStreamWaitEvent(c.sL, ev_tul(k - 1), 0));
      // block row k-1 is final here: its trailing updates and left swaps are complete
      if (sink) CKR((*sink)(grid[k - 1].col0, grid[k - 1].col0 + grid[k - 1].bw, c.sL));
      CKR(left_swaps(k, c.sL));
    }
    if (k + 1 < count) {
      if (k > 0) CK(cudaStreamWaitEvent(c.sP, first_blk ? ev_first(k - 1) : ev_ck(chunk_of_block(k + 1), k - 1), 0));
      CKR(update_cols(k, grid[k + 1].col0, grid[k + 1].col0 + grid[k + 1].bw, c.sP, PFLU_TRACE_TU_L));
      CK(cudaEventRecord(ev_tul(k), c.sP));
      CKR(pf(k + 1, c.sP));
      if (sched == 2 && lo_r < hi_r && grid[k].col0 + grid[k].bw < m) {
        // LA_MB: the panel's SMs rejoin TU_R(k) -- a join grid on the same tile queue (it runs once
        // U12 of step k is solved; ev_pf(k+1), recorded after it, orders every later reader)
        CK(cudaStreamWaitEvent(c.sP, c.swev[k], 0));
        bool done = false;
        CKR(tur_gemm_pers(k, lo_r, hi_r, true, c.sP, &done));
      }
      CK(cudaEventRecord(ev_pf(k + 1), c.sP));
    } else {
      CK(cudaEventRecord(ev_tul(k), c.sP));
    }
  }
  CK(cudaEventRecord(c.ev[1], c.sP));
  CK(cudaStreamWaitEvent(user, c.ev[1], 0));
  for (int ch = 0; ch < nch; ++ch) {
    CK(cudaEventRecord(ev_ck(ch, count - 1), c.sC[ch]));
    CK(cudaStreamWaitEvent(user, ev_ck(ch, count - 1), 0));
  }
  CK(cudaEventRecord(ev_tul(count - 1), c.sL));
  CK(cudaStreamWaitEvent(user, ev_tul(count - 1), 0));
  return PFLU_OK;
}

static int check_dims(int64_t m, int64_t n, int64_t lda, int64_t b, int lookahead) {
  if (m < 1) return -2;
  if (n < 1 || n > m) return -3;
  if (lda < n) return -4;
  if (b < 1) return -5;
  if (lookahead != 0 && lookahead != 1) return -6;
  if (std::min(b, n) > PLAN_MAX) return set_err(PFLU_ERR_UNSUPPORTED, "block size %lld > %d", (long long)b, PLAN_MAX);
  return PFLU_OK;
}

static int finish_info(DevCtx& c, cudaStream_t st, int64_t* info) {
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, c.info, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (info) *info = (h == ~0ull) ? 0 : (int64_t)h;
  return PFLU_OK;
}

}  // namespace pflu

#include "pflu_mg.cuh"
#include "pflu_qr.cuh"

using namespace pflu;

// ==========================================================================================
// C ABI

extern "C" {

int pflu_version(void) { return 1; }

long long pflu_launch_count(void) { return g_launches.load(); }
unsigned pflu_set_trace_mask(unsigned mask) {
  const unsigned old = g_trace_mask.exchange(mask);
  return old;
}

// Developer hook (not in pflu.h): per-phase clock64 totals of the panel kernel's CTA 0.
int pflu_debug_panel_profile(void* dev_buf) {
  g_prof = (unsigned long long*)dev_buf;
  return PFLU_OK;
}

const char* pflu_last_error(void) { return g_err.c_str(); }

void pflu_default_options(pflu_options* opt) {
  if (!opt) return;
  memset(opt, 0, sizeof(*opt));
}

int pflu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int pflu_getrf_device(double* d_a, int64_t m, int64_t n, int64_t lda, int64_t b, int lookahead, int64_t* d_ipiv,
                      int64_t* info, void* stream, const pflu_options* opt_in, pflu_trace_event* trace, int trace_cap,
                      int* trace_len) {
  if (!d_a) return -1;
  CKR(check_dims(m, n, lda, b, lookahead));
  if (!d_ipiv) return -7;
  pflu_options opt;
  pflu_default_options(&opt);
  if (opt_in) opt = *opt_in;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  cudaStream_t st = (cudaStream_t)stream;
  Tracer tr;
  tr.c = c;
  tr.on = trace != nullptr && trace_cap > 0;
  CKR(getrf_async(*c, d_a, m, n, lda, std::min(b, n), lookahead, d_ipiv, c->info, st, opt, tr));
  CKR(finish_info(*c, st, info));
  return tr.collect(trace, trace_cap, trace_len);
}

// Host-buffer factorization: H2D, the blocked factorization, and a D2H that streams every block
// row to the host as soon as it is final (overlapping the rest of the run); the remaining rows and
// the pivots follow the last step.
static int getrf_host_impl(double* a, int64_t m, int64_t n, int64_t lda, int64_t b, int lookahead, int64_t* ipiv,
                           int64_t* info, const pflu_options& opt) {
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  // device copy (grow-only workspace kept across calls; pflu_release_workspace frees it) with an
  // even leading dimension (16-byte aligned rows for the vector paths)
  const int64_t ldd = (n + 1) & ~(int64_t)1;
  const size_t need = (size_t)m * ldd;
  if (c->hbuf_cap < need) {
    if (c->hbuf) CK(cudaFree(c->hbuf));
    c->hbuf = nullptr;
    c->hbuf_cap = 0;
    if (cudaMalloc(&c->hbuf, sizeof(double) * need) != cudaSuccess) {
      cudaGetLastError();
      return set_err(PFLU_ERR_NOMEM, "cudaMalloc of the %zu-byte device copy failed", sizeof(double) * need);
    }
    c->hbuf_cap = need;
  }
  if (c->hpiv_cap < (size_t)n) {
    if (c->hpiv) CK(cudaFree(c->hpiv));
    c->hpiv = nullptr;
    c->hpiv_cap = 0;
    if (cudaMalloc(&c->hpiv, sizeof(int64_t) * n) != cudaSuccess) {
      cudaGetLastError();
      return set_err(PFLU_ERR_NOMEM, "cudaMalloc pivots failed");
    }
    c->hpiv_cap = n;
  }
  double* d_a = c->hbuf;
  int64_t* d_piv = c->hpiv;
  cudaStream_t st = c->sH, sD = c->sD;
  static const bool timing = getenv("PFLU_HOST_TIMING") != nullptr;  // developer: split of the call
  cudaEvent_t t0 = nullptr, t1 = nullptr, t2 = nullptr, t3 = nullptr;
  if (timing) {
    for (cudaEvent_t* e : {&t0, &t1, &t2, &t3}) CK(cudaEventCreate(e));
    CK(cudaEventRecord(t0, st));
  }
  HostIn hin{a, lda, g_h2d_chunks};
  const bool chunked_in = lookahead == 1 && g_h2d_chunks > 1;
  if (!chunked_in && cudaMemcpy2DAsync(d_a, ldd * 8, a, lda * 8, n * 8, m, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return set_err(PFLU_ERR_CUDA, "H2D copy failed");
  if (timing) CK(cudaEventRecord(t1, st));
  int64_t sent = 0;
  size_t nev = 0;
  auto next_event = [&](cudaEvent_t* e) -> int {
    while (c->rev.size() <= nev) {
      cudaEvent_t x;
      CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
      c->rev.push_back(x);
    }
    *e = c->rev[nev++];
    return PFLU_OK;
  };
  RowSink sink = [&](int64_t r0, int64_t r1, cudaStream_t after) -> int {
    if (r0 != sent || r1 <= r0) return PFLU_OK;
    cudaEvent_t e;
    CKR(next_event(&e));
    CK(cudaEventRecord(e, after));
    CK(cudaStreamWaitEvent(sD, e, 0));
    CK(cudaMemcpy2DAsync(a + r0 * lda, lda * 8, d_a + r0 * ldd, ldd * 8, n * 8, r1 - r0, cudaMemcpyDeviceToHost, sD));
    sent = r1;
    return PFLU_OK;
  };
  Tracer tr;
  tr.c = c;
  tr.on = false;
  CKR(getrf_async(*c, d_a, m, n, ldd, std::min(b, n), lookahead, d_piv, c->info, st, opt, tr, &sink,
                  chunked_in ? &hin : nullptr));
  if (timing) CK(cudaEventRecord(t2, st));
  cudaEvent_t e;
  CKR(next_event(&e));
  CK(cudaEventRecord(e, st));
  CK(cudaStreamWaitEvent(sD, e, 0));
  if (sent < m)
    CK(cudaMemcpy2DAsync(a + sent * lda, lda * 8, d_a + sent * ldd, ldd * 8, n * 8, m - sent, cudaMemcpyDeviceToHost, sD));
  CK(cudaMemcpyAsync(ipiv, d_piv, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, sD));
  CKR(finish_info(*c, st, info));
  CK(cudaStreamSynchronize(sD));
  if (timing) {
    CK(cudaEventRecord(t3, sD));
    CK(cudaEventSynchronize(t3));
    float h2d = 0, fac = 0, tail = 0;
    cudaEventElapsedTime(&h2d, t0, t1);
    cudaEventElapsedTime(&fac, t1, t2);
    cudaEventElapsedTime(&tail, t2, t3);
    fprintf(stderr, "pflu_getrf: H2D %.1f ms, factorization %.1f ms, D2H after the last step %.1f ms\n", h2d, fac, tail);
    for (cudaEvent_t x : {t0, t1, t2, t3}) cudaEventDestroy(x);
  }
  return PFLU_OK;
}

int pflu_getrf(double* a, int64_t m, int64_t n, int64_t lda, int64_t b, int lookahead, int64_t* ipiv, int64_t* info,
               const pflu_options* opt) {
  if (!a) return -1;
  CKR(check_dims(m, n, lda, b, lookahead));
  if (!ipiv) return -7;
  pflu_options o;
  pflu_default_options(&o);
  if (opt) o = *opt;
  const int rc = getrf_host_impl(a, m, n, lda, b, lookahead, ipiv, info, o);
  if (rc != PFLU_OK) cudaGetLastError();
  return rc;
}

int pflu_init(int n_gpus, const int* devices) {
  if (n_gpus < 1 || n_gpus > 64) return -1;
  std::lock_guard<std::mutex> lk(g_mu);
  const int rc = mg_init(n_gpus, devices);
  if (rc != PFLU_OK) cudaGetLastError();
  return rc;
}

int pflu_finalize(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return mg_finalize();
}

int pflu_mg_size(void) { return g_mg.P; }
int pflu_mg_uses_nccl(void) { return g_mg.nccl ? 1 : 0; }

int64_t pflu_mg_local_cols(int64_t n, int64_t b, int n_gpus, int rank) {
  if (n < 0 || b < 1 || n_gpus < 1 || rank < 0 || rank >= n_gpus) return -1;
  return mg_local_cols(n, b, n_gpus, rank);
}

int pflu_getrf_mg(double* a, int64_t n, int64_t lda, int64_t b, int lookahead, int n_gpus, int64_t* ipiv,
                  int64_t* info, const pflu_options* opt, pflu_trace_event* trace, int trace_cap, int* trace_len) {
  if (!a) return -1;
  if (n < 1) return -2;
  if (lda < n) return -3;
  if (b < 1) return -4;
  if (lookahead != 0 && lookahead != 1) return -5;
  if (n_gpus < 1 || n_gpus > 64) return -6;
  if (!ipiv) return -7;
  if (std::min(b, n) > PLAN_MAX) return set_err(PFLU_ERR_UNSUPPORTED, "block size %lld > %d", (long long)b, PLAN_MAX);
  pflu_options o;
  pflu_default_options(&o);
  if (opt) o = *opt;
  static const bool force = getenv("PFLU_MG_FORCE") && atoi(getenv("PFLU_MG_FORCE")) != 0;
  if (trace_len) *trace_len = 0;
  if (n_gpus == 1 && !force) {
    const int rc = getrf_host_impl(a, n, n, lda, b, lookahead, ipiv, info, o);
    if (rc != PFLU_OK) cudaGetLastError();
    return rc;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  int dev0 = 0;
  cudaGetDevice(&dev0);
  const int rc = mg_getrf(a, n, lda, b, lookahead, n_gpus, ipiv, info, o, trace, trace_cap, trace_len);
  cudaSetDevice(dev0);
  if (rc != PFLU_OK) cudaGetLastError();
  return rc;
}

int pflu_release_workspace(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  CK(cudaDeviceSynchronize());
  if (c->hbuf) CK(cudaFree(c->hbuf));
  if (c->hpiv) CK(cudaFree(c->hpiv));
  c->hbuf = nullptr;
  c->hpiv = nullptr;
  c->hbuf_cap = c->hpiv_cap = 0;
  g_qr[c->dev].release();
  return PFLU_OK;
}

int pflu_panel(double* d_a, int64_t lda, int64_t m, int64_t d, int64_t col, int64_t w, int64_t* d_ipiv, int64_t* info,
               void* stream, const pflu_options* opt_in) {
  if (!d_a) return -1;
  if (lda < 1) return -2;
  if (m < 1) return -3;
  if (d < 0 || d >= m) return -4;
  if (col < 0 || col + w > lda) return -5;
  if (w < 1) return -6;
  if (!d_ipiv) return -7;
  pflu_options opt;
  pflu_default_options(&opt);
  if (opt_in) opt = *opt_in;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  cudaStream_t st = (cudaStream_t)stream;
  if (!info) return panel_factor(*c, d_a, lda, m, d, col, w, d_ipiv, c->info, opt, st);  // asynchronous
  CK(cudaMemsetAsync(c->info, 0xff, 8, st));
  CKR(panel_factor(*c, d_a, lda, m, d, col, w, d_ipiv, c->info, opt, st));
  return finish_info(*c, st, info);
}

int pflu_copy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t height,
                void* stream) {
  if (!dst) return -1;
  if (dpitch < width) return -2;
  if (!src) return -3;
  if (spitch < width) return -4;
  if (width < 0) return -5;
  if (height < 0) return -6;
  if (width == 0 || height == 0) return PFLU_OK;
  CK(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width, (size_t)height, cudaMemcpyDefault,
                       (cudaStream_t)stream));
  return PFLU_OK;
}

int pflu_info_reset(void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  CK(cudaMemsetAsync(c->info, 0xff, 8, (cudaStream_t)stream));
  return PFLU_OK;
}

int pflu_info_read(int64_t* info, void* stream) {
  if (!info) return -1;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  return finish_info(*c, (cudaStream_t)stream, info);
}

int pflu_pivot_plan(const int64_t* d_ipiv, int64_t d, int64_t nb, int64_t* d_plan, void* stream) {
  if (!d_ipiv) return -1;
  if (d < 0) return -2;
  if (nb < 1 || nb > PLAN_MAX) return -3;
  if (!d_plan) return -4;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  return launch_plan(d_ipiv, d, (int)nb, d_plan, (cudaStream_t)stream);
}

int pflu_swap_trsm_plan(double* d_a, int64_t lda, int64_t d, int64_t nb, const int64_t* d_plan, int64_t c0,
                        int64_t c1, const double* d_l, int64_t ldl, void* stream) {
  if (!d_a) return -1;
  if (lda < 1) return -2;
  if (d < 0) return -3;
  if (nb < 1 || nb > PLAN_MAX) return -4;
  if (!d_plan) return -5;
  if (c0 < 0) return -6;
  if (c1 < c0 || c1 > lda) return -7;
  if (d_l && ldl < nb) return -9;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  return launch_swap(d_a, lda, d, (int)nb, d_plan, c0, c1, d_l, ldl, d_l != nullptr, (cudaStream_t)stream);
}

int pflu_diag_inv(const double* d_l, int64_t ldl, int64_t nb, double* d_inv, void* stream) {
  if (!d_l) return -1;
  if (nb < 1 || nb > PLAN_MAX) return -3;
  if (ldl < nb) return -2;
  if (!d_inv) return -4;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  return launch_diag_inv(d_l, ldl, (int)nb, d_inv, (cudaStream_t)stream);
}

int pflu_swap_trsm_inv(double* d_a, int64_t lda, int64_t d, int64_t nb, const int64_t* d_plan, int64_t c0,
                       int64_t c1, const double* d_l, int64_t ldl, const double* d_inv, void* stream) {
  if (!d_a) return -1;
  if (lda < 1) return -2;
  if (d < 0) return -3;
  if (nb < 1 || nb > PLAN_MAX) return -4;
  if (!d_plan) return -5;
  if (c0 < 0) return -6;
  if (c1 < c0 || c1 > lda) return -7;
  if (!d_l) return -8;
  if (ldl < nb) return -9;
  if (!d_inv) return -10;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  return launch_swap(d_a, lda, d, (int)nb, d_plan, c0, c1, d_l, ldl, true, (cudaStream_t)stream, nb <= 512 ? d_inv : nullptr);
}

int pflu_laswp(double* d_a, int64_t lda, int64_t c0, int64_t c1, const int64_t* d_ipiv, int64_t k1, int64_t k2,
               void* stream) {
  if (!d_a) return -1;
  if (lda < 1) return -2;
  if (c0 < 0 || c0 > lda) return -3;
  if (c1 < c0 || c1 > lda) return -4;
  if (!d_ipiv) return -5;
  if (k1 < 0) return -6;
  if (k2 < k1) return -7;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  cudaStream_t st = (cudaStream_t)stream;
  for (int64_t k = k1; k < k2; k += PLAN_MAX) {
    int np = (int)std::min<int64_t>(PLAN_MAX, k2 - k);
    CKR(launch_plan(d_ipiv, k, np, c->plan[0], st));
    CKR(launch_swap(d_a, lda, k, np, c->plan[0], c0, c1, nullptr, lda, false, st));
  }
  return PFLU_OK;
}

int pflu_swap_trsm(double* d_a, int64_t lda, int64_t d, int64_t lcol, int64_t nb, const int64_t* d_ipiv, int64_t c0,
                   int64_t c1, void* stream) {
  if (!d_a) return -1;
  if (lda < 1) return -2;
  if (d < 0) return -3;
  if (lcol < 0) return -4;
  if (nb < 1 || nb > PLAN_MAX) return -5;
  if (!d_ipiv) return -6;
  if (c0 < 0) return -7;
  if (c1 < c0 || c1 > lda) return -8;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  cudaStream_t st = (cudaStream_t)stream;
  CKR(launch_plan(d_ipiv, d, (int)nb, c->plan[0], st));
  return launch_swap(d_a, lda, d, (int)nb, c->plan[0], c0, c1, d_a + d * lda + lcol, lda, true, st);
}

int pflu_trsm(const double* d_l, int64_t ldl, int64_t nb, double* d_x, int64_t ldx, int64_t ncols, void* stream) {
  if (!d_l) return -1;
  if (ldl < nb) return -2;
  if (nb < 0 || nb > PLAN_MAX) return -3;
  if (!d_x) return -4;
  if (ldx < ncols) return -5;
  if (ncols < 0) return -6;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  return launch_trsm(d_l, ldl, (int)nb, d_x, ldx, ncols, (cudaStream_t)stream);
}

int pflu_gemm_update(double* d_c, int64_t ldc, const double* d_a, int64_t lda, const double* d_b, int64_t ldb,
                     int64_t m, int64_t n, int64_t k, int exact, void* stream) {
  if (!d_c) return -1;
  if (ldc < n) return -2;
  if (!d_a) return -3;
  if (lda < k) return -4;
  if (!d_b) return -5;
  if (ldb < n) return -6;
  if (m < 0) return -7;
  if (n < 0) return -8;
  if (k < 0) return -9;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  return launch_gemm(d_c, ldc, d_a, lda, d_b, ldb, m, n, k, exact != 0, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------------------------
// Householder QR (Kind.QR)

static int check_qr_dims(int64_t m, int64_t n, int64_t lda, int64_t b, int lookahead) {
  if (m < 1) return -2;
  if (n < 1 || n > m) return -3;
  if (lda < n) return -4;
  if (b < 1) return -5;
  if (lookahead != 0 && lookahead != 1) return -6;
  if (std::min(b, n) > 1024) return set_err(PFLU_ERR_UNSUPPORTED, "QR block size %lld > 1024", (long long)b);
  return PFLU_OK;
}

int pflu_geqrf_device(double* d_a, int64_t m, int64_t n, int64_t lda, int64_t b, int lookahead, double* d_tau,
                      void* stream, pflu_trace_event* trace, int trace_cap, int* trace_len) {
  if (!d_a) return -1;
  CKR(check_qr_dims(m, n, lda, b, lookahead));
  if (!d_tau) return -7;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  cudaStream_t st = (cudaStream_t)stream;
  Tracer tr;
  tr.c = c;
  tr.on = trace != nullptr && trace_cap > 0;
  CKR(geqrf_async(*c, d_a, m, n, lda, std::min(b, n), lookahead, d_tau, st, nullptr, &tr));
  CK(cudaStreamSynchronize(st));
  return tr.collect(trace, trace_cap, trace_len);
}

// Host buffers: H2D into the grow-only device copy shared with pflu_getrf, the factorization, and a
// D2H that streams every row block as soon as it is final (overlapping the rest of the run).
int pflu_geqrf(double* a, int64_t m, int64_t n, int64_t lda, int64_t b, int lookahead, double* tau) {
  if (!a) return -1;
  CKR(check_qr_dims(m, n, lda, b, lookahead));
  if (!tau) return -7;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  QrCtx* q = nullptr;
  CKR(qr_ctx(*c, &q));
  const int64_t ldd = qr_even(n);
  const size_t need = (size_t)m * ldd;
  if (c->hbuf_cap < need) {
    if (c->hbuf) CK(cudaFree(c->hbuf));
    c->hbuf = nullptr;
    c->hbuf_cap = 0;
    if (cudaMalloc(&c->hbuf, sizeof(double) * need) != cudaSuccess) {
      cudaGetLastError();
      return set_err(PFLU_ERR_NOMEM, "pflu_geqrf: device copy of %lld x %lld", (long long)m, (long long)n);
    }
    c->hbuf_cap = need;
  }
  CKR(q->htau.need((size_t)n));
  double* d_a = c->hbuf;
  double* d_tau = q->htau.p;
  cudaStream_t st = c->sH, sD = c->sD;
  static const int qr_chunks = []() { const char* e = getenv("PFLU_QR_H2D_CHUNKS"); return e ? atoi(e) : 6; }();
  const bool chunked = lookahead == 1 && qr_chunks > 1 && std::min(b, n) < n;
  if (!chunked && cudaMemcpy2DAsync(d_a, ldd * 8, a, lda * 8, n * 8, m, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return set_err(PFLU_ERR_CUDA, "pflu_geqrf: H2D failed");
  int64_t sent = 0;
  size_t nev = 0;
  auto next_event = [&](cudaEvent_t* e) -> int {
    while (c->rev.size() <= nev) {
      cudaEvent_t x;
      CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
      c->rev.push_back(x);
    }
    *e = c->rev[nev++];
    return PFLU_OK;
  };
  RowSink sink = [&](int64_t r0, int64_t r1, cudaStream_t after) -> int {
    if (r0 != sent || r1 <= r0) return PFLU_OK;
    cudaEvent_t e;
    CKR(next_event(&e));
    CK(cudaEventRecord(e, after));
    CK(cudaStreamWaitEvent(sD, e, 0));
    CK(cudaMemcpy2DAsync(a + r0 * lda, lda * 8, d_a + r0 * ldd, ldd * 8, n * 8, r1 - r0, cudaMemcpyDeviceToHost, sD));
    sent = r1;
    return PFLU_OK;
  };
  if (chunked) {
    RowSinkM sinkm = [&](int64_t r0, int64_t r1, const std::vector<cudaEvent_t>& after) -> int {
      if (r0 != sent || r1 <= r0) return PFLU_OK;
      for (cudaEvent_t ev : after) CK(cudaStreamWaitEvent(sD, ev, 0));
      CK(cudaMemcpy2DAsync(a + r0 * lda, lda * 8, d_a + r0 * ldd, ldd * 8, n * 8, r1 - r0, cudaMemcpyDeviceToHost, sD));
      sent = r1;
      return PFLU_OK;
    };
    CKR(geqrf_host_chunked(*c, d_a, m, n, ldd, std::min(b, n), d_tau, st, a, lda, qr_chunks, sinkm));
  } else {
    CKR(geqrf_async(*c, d_a, m, n, ldd, std::min(b, n), lookahead, d_tau, st, &sink));
  }
  cudaEvent_t e;
  CKR(next_event(&e));
  CK(cudaEventRecord(e, st));
  CK(cudaStreamWaitEvent(sD, e, 0));
  if (sent < m)
    CK(cudaMemcpy2DAsync(a + sent * lda, lda * 8, d_a + sent * ldd, ldd * 8, n * 8, m - sent, cudaMemcpyDeviceToHost, sD));
  CK(cudaMemcpyAsync(tau, d_tau, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, sD));
  CK(cudaStreamSynchronize(sD));
  CK(cudaStreamSynchronize(st));
  return PFLU_OK;
}

int pflu_qr_panel(double* d_a, int64_t lda, int64_t m, int64_t d, int64_t col, int64_t w, double* d_tau, void* stream) {
  if (!d_a) return -1;
  if (lda < col + w || col < 0) return -2;
  if (m < 1) return -3;
  if (d < 0 || d >= m) return -4;
  if (w < 1 || w > m - d) return -6;
  if (!d_tau) return -7;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  QrCtx* q = nullptr;
  CKR(qr_ctx(*c, &q));
  CKR(qr_panel(*c, *q, d_a, lda, m, d, col, w, d_tau, q->leaf, (cudaStream_t)stream));
  return PFLU_OK;
}

int pflu_larft(const double* d_v, int64_t ldv, int64_t mp, int64_t k, const double* d_tau, double* d_t, int64_t ldt,
               void* stream) {
  if (!d_v) return -1;
  if (ldv < k) return -2;
  if (mp < k) return -3;
  if (k < 1 || k > 1024) return -4;
  if (!d_tau) return -5;
  if (!d_t) return -6;
  if (ldt < k) return -7;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  QrCtx* q = nullptr;
  CKR(qr_ctx(*c, &q));
  cudaStream_t st = (cudaStream_t)stream;
  QrSlot& sl = q->slot(st);
  // the panel view: rows [0, mp) of columns [0, k) at d_v
  CKR(qr_build(*c, sl.ws, sl.refl, d_v, ldv, 0, mp, 0, (int)k, d_tau, st));
  // T = (T^T)^T into the caller's upper-triangular layout
  std::vector<double> tt((size_t)(k * sl.refl.ldt)), t((size_t)(k * ldt), 0.0);
  CK(cudaMemcpyAsync(tt.data(), sl.refl.tt.p, sizeof(double) * tt.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(t.data(), d_t, sizeof(double) * t.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < k; ++i)
    for (int64_t j = 0; j < k; ++j) t[(size_t)(i * ldt + j)] = j >= i ? tt[(size_t)(j * sl.refl.ldt + i)] : 0.0;
  CK(cudaMemcpyAsync(d_t, t.data(), sizeof(double) * t.size(), cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  return PFLU_OK;
}

int pflu_apply_block_reflector(const double* d_v, int64_t ldv, int64_t mp, int64_t k, const double* d_tau, double* d_c,
                               int64_t ldc, int64_t nc, void* stream) {
  if (!d_v) return -1;
  if (ldv < k) return -2;
  if (mp < k) return -3;
  if (k < 1 || k > 1024) return -4;
  if (!d_tau) return -5;
  if (!d_c) return -6;
  if (ldc < nc) return -7;
  if (nc < 0) return -8;
  std::lock_guard<std::mutex> lk(g_mu);
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  QrCtx* q = nullptr;
  CKR(qr_ctx(*c, &q));
  cudaStream_t st = (cudaStream_t)stream;
  QrSlot& sl = q->slot(st);
  CKR(qr_build(*c, sl.ws, sl.refl, d_v, ldv, 0, mp, 0, (int)k, d_tau, st));
  CKR(qr_apply(*c, sl.ws, qr_view(sl.refl), d_c, ldc, nc, st));
  return PFLU_OK;
}

}  // extern "C"
