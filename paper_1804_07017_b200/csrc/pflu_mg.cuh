// pflu_mg.cuh -- multi-GPU LU behind the C ABI (pflu_init / pflu_finalize / pflu_getrf_mg).
//
// the reference's in-process drop-in call (dmf_la, factor.py:455-515) reaching
// several GPUs without a process launcher.  ONE process drives P devices, one host thread per rank:
//
//   * 1-D block-cyclic columns: global column block j (width b) lives on rank j % P, stored
//     contiguously (n x nloc row-major, even leading dimension); rows are not distributed, so the
//     row interchanges of partial pivoting stay local;
//   * per step k the owner o = k % P factors its copy of block k (the single-GPU panel kernels), packs
//     rows [kb, n) of it and the step's pivots into ONE message, and every rank receives it: NCCL
//     ncclBroadcast (communicators from ncclCommInitAll) or, when two ranks share a device (tests on
//     one GPU) or PFLU_MG_TRANSPORT=copy, device-to-device / peer copies ordered by events;
//   * every rank then runs the pivot plan, the fused swap + U12 solve (L11 from the message) and the
//     DMMA GEMM (L21 from the message) on its own trailing columns; the deferred left swaps on its
//     columns left of the panel;
//   * look-ahead 1 across ranks (dmf_la): the owner of block k+1 first updates that block (TU_L) and
//     factors / sends it on the high-priority panel stream while every rank runs the rest of TU_R(k)
//     on its update stream.
//
// The schedule is the one of paper_1804_07017_b200/dist.py (the torch.distributed driver, one process
// per GPU), written against the same kernels.  NCCL is loaded with dlopen at pflu_init time, so
// libpflu.so has no link-time NCCL dependency (the process's NCCL, e.g. the one torch loaded, is used).
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <thread>

namespace pflu {

// ---- NCCL entry points (dlopen)
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  bool load() {
    if (h) return true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    commInitAll = (decltype(commInitAll))dlsym(h, "ncclCommInitAll");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    broadcast = (decltype(broadcast))dlsym(h, "ncclBroadcast");
    errorString = (decltype(errorString))dlsym(h, "ncclGetErrorString");
    return commInitAll && commDestroy && broadcast && errorString;
  }
};
static NcclApi g_nccl;

#define NCK(expr)                                                                                 \
  do {                                                                                            \
    ncclResult_t _n = (expr);                                                                     \
    if (_n != ncclSuccess)                                                                        \
      return set_err(PFLU_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, g_nccl.errorString(_n),       \
                     __FILE__, __LINE__);                                                         \
  } while (0)

// ---- block-cyclic bookkeeping (host; also exported for the CPU tests)
static inline int64_t mg_nblocks(int64_t n, int64_t b) { return (n + b - 1) / b; }
static inline int64_t mg_local_cols(int64_t n, int64_t b, int P, int r) {
  int64_t s = 0;
  for (int64_t j = r; j < mg_nblocks(n, b); j += P) s += std::min(b, n - j * b);
  return s;
}
static inline int64_t mg_local_cols_before(int64_t k, int64_t n, int64_t b, int P, int r) {
  int64_t s = 0;
  for (int64_t j = r; j < std::min(k, mg_nblocks(n, b)); j += P) s += std::min(b, n - j * b);
  return s;
}

struct MgRank {
  int r = 0, dev = 0;
  cudaStream_t sP = nullptr, sU = nullptr;
  double* a = nullptr;  // n x ld local columns
  size_t a_cap = 0;
  double* msg[2] = {nullptr, nullptr};  // packed panel ((n - kb) x bw) + bw pivots (int64 bits)
  size_t msg_cap = 0;
  int64_t* piv = nullptr;
  size_t piv_cap = 0;
  int64_t* plans = nullptr;  // per step: 1 + 3 b words
  double* invs = nullptr;    // per step: inverted 32x32 diagonal blocks (fast mode)
  size_t plans_cap = 0, invs_cap = 0;
  unsigned long long* info = nullptr;
  std::vector<cudaEvent_t> ev;   // [k][0] message ready (plan done), [k][1] TU_R(k) + left swaps done,
                                 // [k][2] packed (owner, copy transport)
  std::vector<cudaEvent_t> tev;  // rank 0 tracing
  std::atomic<int64_t> packed{-1}, received{-1};  // host: last step whose event was recorded
};

struct MgCtx {
  int P = 0;
  std::vector<int> devs;
  bool nccl = false;
  std::vector<ncclComm_t> comms;
  std::vector<std::unique_ptr<MgRank>> ranks;
};
static MgCtx g_mg;
static std::string g_mg_transport = []() { const char* e = getenv("PFLU_MG_TRANSPORT"); return std::string(e ? e : ""); }();

static int mg_release_ranks() {
  for (auto& R : g_mg.ranks) {
    if (!R) continue;
    CK(cudaSetDevice(R->dev));
    CK(cudaDeviceSynchronize());
    for (double* p : {R->a, R->msg[0], R->msg[1], R->invs})
      if (p) CK(cudaFree(p));
    if (R->piv) CK(cudaFree(R->piv));
    if (R->plans) CK(cudaFree(R->plans));
    if (R->info) CK(cudaFree(R->info));
    for (cudaEvent_t e : R->ev) CK(cudaEventDestroy(e));
    for (cudaEvent_t e : R->tev) CK(cudaEventDestroy(e));
    if (R->sP) CK(cudaStreamDestroy(R->sP));
    if (R->sU) CK(cudaStreamDestroy(R->sU));
  }
  g_mg.ranks.clear();
  return PFLU_OK;
}

static int mg_finalize() {
  CKR(mg_release_ranks());
  if (g_mg.nccl)
    for (ncclComm_t c : g_mg.comms) NCK(g_nccl.commDestroy(c));
  g_mg.comms.clear();
  g_mg.nccl = false;
  g_mg.P = 0;
  g_mg.devs.clear();
  return PFLU_OK;
}

static int mg_init(int P, const int* devices) {
  if (g_mg.P == P) {
    bool same = true;
    for (int r = 0; r < P; ++r) same = same && g_mg.devs[r] == (devices ? devices[r] : r);
    if (same) return PFLU_OK;
  }
  CKR(mg_finalize());
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  g_mg.devs.resize(P);
  bool distinct = true;
  for (int r = 0; r < P; ++r) {
    const int d = devices ? devices[r] : r;
    if (d < 0 || d >= ndev) {
      g_mg.devs.clear();
      return set_err(PFLU_ERR_UNSUPPORTED, "rank %d: device %d requested, %d visible", r, d, ndev);
    }
    for (int q = 0; q < r; ++q) distinct = distinct && g_mg.devs[q] != d;
    g_mg.devs[r] = d;
  }
  // NCCL needs one device per rank; ranks sharing a device (single-GPU tests) use the copy transport
  g_mg.nccl = distinct && g_mg_transport != "copy";
  if (g_mg.nccl) {
    if (!g_nccl.load()) {
      g_mg.devs.clear();
      return set_err(PFLU_ERR_UNSUPPORTED, "libnccl.so.2 not found (dlopen): cannot run %d GPUs", P);
    }
    g_mg.comms.resize(P);
    NCK(g_nccl.commInitAll(g_mg.comms.data(), P, g_mg.devs.data()));
  }
  for (int r = 0; r < P; ++r) {
    auto R = std::make_unique<MgRank>();
    R->r = r;
    R->dev = g_mg.devs[r];
    CK(cudaSetDevice(R->dev));
    DevCtx* c = nullptr;
    CKR(ctx_get(&c));
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&R->sP, cudaStreamNonBlocking, hi));
    CK(cudaStreamCreateWithPriority(&R->sU, cudaStreamNonBlocking, lo));
    CK(cudaMalloc(&R->info, 64));
    g_mg.ranks.push_back(std::move(R));
  }
  // peer access between distinct devices (copy transport over NVLink)
  if (!g_mg.nccl)
    for (int r = 0; r < P; ++r)
      for (int q = 0; q < P; ++q)
        if (g_mg.devs[r] != g_mg.devs[q]) {
          int can = 0;
          CK(cudaDeviceCanAccessPeer(&can, g_mg.devs[r], g_mg.devs[q]));
          if (can) {
            CK(cudaSetDevice(g_mg.devs[r]));
            cudaError_t e = cudaDeviceEnablePeerAccess(g_mg.devs[q], 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
            cudaGetLastError();
          }
        }
  g_mg.P = P;
  return PFLU_OK;
}

template <class T>
static int mg_grow(T** p, size_t* cap, size_t need) {
  if (*cap >= need) return PFLU_OK;
  if (*p) CK(cudaFree(*p));
  *p = nullptr;
  *cap = 0;
  if (cudaMalloc(p, sizeof(T) * std::max<size_t>(need, 1)) != cudaSuccess) {
    cudaGetLastError();
    return set_err(PFLU_ERR_NOMEM, "cudaMalloc of %zu bytes failed", sizeof(T) * need);
  }
  *cap = need;
  return PFLU_OK;
}

struct MgJob {
  double* a;  // host, n x n, leading dimension lda
  int64_t n, lda, b;
  int lookahead;
  pflu_options opt;
  int64_t* ipiv;  // host
  std::vector<int64_t> info;
  std::vector<int> rc;
  std::vector<std::string> err;
  pflu_trace_event* trace;
  int trace_cap;
  int trace_len;
};

static void mg_wait_flag(const std::atomic<int64_t>& f, int64_t k) {
  while (f.load(std::memory_order_acquire) < k) std::this_thread::yield();
}

// one rank's whole factorization (runs on its own host thread)
static int mg_rank_run(MgRank& R, MgJob& J) {
  const int P = g_mg.P, r = R.r;
  const int64_t n = J.n, b = J.b;
  const int count = (int)mg_nblocks(n, b);
  const bool exact = J.opt.exact != 0;
  CK(cudaSetDevice(R.dev));
  DevCtx* c = nullptr;
  CKR(ctx_get(&c));
  const int64_t nloc = mg_local_cols(n, b, P, r);
  const int64_t ld = std::max<int64_t>(2, (nloc + 1) & ~(int64_t)1);
  const int64_t bb = std::min(b, n);
  CKR(mg_grow(&R.a, &R.a_cap, (size_t)n * ld));
  size_t msg_need = (size_t)n * bb + bb;
  if (R.msg_cap < msg_need) {
    for (double*& m : R.msg) {
      if (m) CK(cudaFree(m));
      m = nullptr;
    }
    R.msg_cap = 0;
    for (double*& m : R.msg)
      if (cudaMalloc(&m, sizeof(double) * msg_need) != cudaSuccess) {
        cudaGetLastError();
        return set_err(PFLU_ERR_NOMEM, "cudaMalloc of the panel message failed");
      }
    R.msg_cap = msg_need;
  }
  CKR(mg_grow(&R.piv, &R.piv_cap, (size_t)n));
  const size_t plan_words = 1 + 3 * (size_t)bb;
  CKR(mg_grow(&R.plans, &R.plans_cap, plan_words * count));
  const bool use_dinv = !exact && g_trsm_dmma && bb <= 512;
  const size_t inv_words = (size_t)1024 * ((bb + 31) / 32);
  if (use_dinv) CKR(mg_grow(&R.invs, &R.invs_cap, inv_words * count));
  while (R.ev.size() < (size_t)count * 3) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    R.ev.push_back(e);
  }
  auto ev = [&](int k, int i) { return R.ev[(size_t)k * 3 + i]; };
  cudaStream_t sP = R.sP, sU = R.sU;
  // tracing (rank 0): PF / TU_L / TU_R / BCAST records
  const bool tracing = r == 0 && J.trace && J.trace_cap > 0;
  struct TRec { int label, k; cudaEvent_t e0, e1; };
  std::vector<TRec> trecs;
  size_t tused = 0;
  cudaEvent_t t0 = nullptr;
  auto tev = [&](cudaEvent_t* e) -> int {
    if (tused == R.tev.size()) {
      cudaEvent_t x;
      CK(cudaEventCreate(&x));
      R.tev.push_back(x);
    }
    *e = R.tev[tused++];
    return PFLU_OK;
  };
  auto tbegin = [&](int label, int k, cudaStream_t st) -> int {
    if (!tracing) return -1;
    TRec t{label, k, nullptr, nullptr};
    if (tev(&t.e0) != PFLU_OK || tev(&t.e1) != PFLU_OK) return -1;
    cudaEventRecord(t.e0, st);
    trecs.push_back(t);
    return (int)trecs.size() - 1;
  };
  auto tend = [&](int i, cudaStream_t st) {
    if (i >= 0) cudaEventRecord(trecs[i].e1, st);
  };
  if (tracing) {
    CKR(tev(&t0));
    CK(cudaEventRecord(t0, sP));
  }
  // H2D of this rank's column blocks
  {
    int64_t cl = 0;
    for (int64_t j = r; j < count; j += P) {
      const int64_t w = std::min(b, n - j * b);
      CK(cudaMemcpy2DAsync(R.a + cl, ld * 8, J.a + j * b, J.lda * 8, w * 8, n, cudaMemcpyHostToDevice, sP));
      cl += w;
    }
  }
  CK(cudaMemsetAsync(R.info, 0xff, 8, sP));
  CK(cudaMemsetAsync(R.piv, 0, sizeof(int64_t) * n, sP));
  CK(cudaEventRecord(ev(0, 1), sP));
  CK(cudaStreamWaitEvent(sU, ev(0, 1), 0));
  // every step's L11 / L21 come from the received message (at P = 1 only with the NCCL transport,
  // PFLU_MG_FORCE: the one-rank communicator still carries every message)
  const bool via_msg = P > 1 || g_mg.nccl;
  auto cols_before = [&](int64_t k) { return mg_local_cols_before(k, n, b, P, r); };
  auto plan_of = [&](int k) { return R.plans + plan_words * k; };
  auto inv_of = [&](int k) { return R.invs + inv_words * k; };

  // owner: factor block k and pack it; every rank: receive it, pivot plan (+ inverted blocks)
  auto pf_send = [&](int k) -> int {
    const int64_t col0 = (int64_t)k * b, bw = std::min(b, n - col0), rows = n - col0;
    const int o = k % P;
    double* msg = R.msg[k % 2];
    int64_t* mpiv = reinterpret_cast<int64_t*>(msg + rows * bw);
    const int np = (int)std::min(bw, rows);
    if (r == o) {
      const int64_t lc = (int64_t)(k / P) * b;
      int t = tbegin(PFLU_TRACE_PF, k, sP);
      pflu_options popt = J.opt;
      if (popt.panel_kernel == 0 && P >= g_emu_grid_ranks && rows > g_grid_rows) {
        popt.panel_kernel = g_tall_kernel;
        if (g_tall_kernel == 4 && popt.panel_ctas == 0 && g_mc_adapt)
          popt.panel_ctas = tall_panel_ctas(rows, (n - col0 - bw) / P, bw);
      }
      CKR(panel_factor(*c, R.a, ld, n, col0, lc, bw, R.piv, R.info, popt, sP));
      tend(t, sP);
      if (via_msg) {
        CK(cudaMemcpy2DAsync(msg, bw * 8, R.a + col0 * ld + lc, ld * 8, bw * 8, rows, cudaMemcpyDeviceToDevice, sP));
        CK(cudaMemcpyAsync(mpiv, R.piv + col0, 8 * np, cudaMemcpyDeviceToDevice, sP));
      }
    }
    if (via_msg) {
      int t = tbegin(PFLU_TRACE_BCAST, k, sP);
      if (g_mg.nccl) {
        NCK(g_nccl.broadcast(msg, msg, (size_t)(rows * bw + np), ncclDouble, o, g_mg.comms[r], sP));
      } else if (r == o) {
        CK(cudaEventRecord(ev(k, 2), sP));
        R.packed.store(k, std::memory_order_release);
      } else {
        MgRank& O = *g_mg.ranks[o];
        mg_wait_flag(O.packed, k);
        CK(cudaStreamWaitEvent(sP, O.ev[(size_t)k * 3 + 2], 0));
        CK(cudaMemcpyPeerAsync(msg, R.dev, O.msg[k % 2], O.dev, sizeof(double) * (rows * bw + np), sP));
      }
      if (r != o) CK(cudaMemcpyAsync(R.piv + col0, mpiv, 8 * np, cudaMemcpyDeviceToDevice, sP));
      tend(t, sP);
    }
    CKR(launch_plan(R.piv, col0, np, plan_of(k), sP));
    const double* l11 = via_msg ? msg : R.a + col0 * ld + (int64_t)(k / P) * b;
    const int64_t ldl = via_msg ? bw : ld;
    if (use_dinv) CKR(launch_diag_inv(l11, ldl, np, inv_of(k), sP));
    CK(cudaEventRecord(ev(k, 0), sP));
    if (!g_mg.nccl && P > 1) R.received.store(k, std::memory_order_release);
    return PFLU_OK;
  };
  // TU of step k on local columns [c0, c1): swaps + solve (L11 from the message), GEMM with L21
  auto update = [&](int k, int64_t c0, int64_t c1, cudaStream_t st) -> int {
    if (c1 <= c0) return PFLU_OK;
    const int64_t col0 = (int64_t)k * b, bw = std::min(b, n - col0), rows = n - col0;
    const int np = (int)std::min(bw, rows);
    const double* msg = R.msg[k % 2];
    const double* l11 = via_msg ? msg : R.a + col0 * ld + (int64_t)(k / P) * b;
    const int64_t ldl = via_msg ? bw : ld;
    CKR(launch_swap(R.a, ld, col0, np, plan_of(k), c0, c1, l11, ldl, true, st, use_dinv ? inv_of(k) : nullptr));
    if (col0 + bw < n)
      CKR(launch_gemm(R.a + (col0 + bw) * ld + c0, ld, l11 + bw * ldl, ldl, R.a + col0 * ld + c0, ld,
                      n - col0 - bw, c1 - c0, bw, exact, st));
    return PFLU_OK;
  };
  auto left_swaps = [&](int k, cudaStream_t st) -> int {
    const int64_t col0 = (int64_t)k * b, bw = std::min(b, n - col0);
    return launch_swap(R.a, ld, col0, (int)std::min(bw, n - col0), plan_of(k), 0, cols_before(k), nullptr, ld,
                       false, st);
  };
  // copy transport: the owner re-packs buffer k % 2 only after every receiver copied step k - 2
  auto wait_receivers = [&](int k) -> int {
    if (g_mg.nccl || P == 1 || k < 2 || r != k % P) return PFLU_OK;
    for (int q = 0; q < P; ++q) {
      if (q == r) continue;
      MgRank& Q = *g_mg.ranks[q];
      mg_wait_flag(Q.received, k - 2);
      CK(cudaStreamWaitEvent(sP, Q.ev[(size_t)(k - 2) * 3 + 0], 0));
    }
    return PFLU_OK;
  };

  if (J.lookahead == 0) {
    for (int k = 0; k < count; ++k) {
      CKR(wait_receivers(k));
      CKR(pf_send(k));
      int t = tbegin(PFLU_TRACE_TU, k, sP);
      CKR(left_swaps(k, sP));
      CKR(update(k, cols_before(k + 1), nloc, sP));
      tend(t, sP);
    }
  } else {
    CKR(pf_send(0));
    for (int k = 0; k < count; ++k) {
      const bool nxt = k + 1 < count;
      const bool own_next = nxt && (k + 1) % P == r;
      const int64_t lo_r = own_next ? cols_before(k + 2) : cols_before(k + 1);
      CK(cudaStreamWaitEvent(sU, ev(k, 0), 0));
      int t = tbegin(PFLU_TRACE_TU_R, k, sU);
      CKR(update(k, lo_r, nloc, sU));
      CKR(left_swaps(k, sU));
      tend(t, sU);
      CK(cudaEventRecord(ev(k, 1), sU));
      if (nxt) {
        if (k > 0) CK(cudaStreamWaitEvent(sP, ev(k - 1, 1), 0));  // message buffer (k+1) % 2 is free
        if (own_next) {
          int tl = tbegin(PFLU_TRACE_TU_L, k, sP);
          CKR(update(k, cols_before(k + 1), cols_before(k + 2), sP));
          tend(tl, sP);
        }
        CKR(wait_receivers(k + 1));
        CKR(pf_send(k + 1));
      }
    }
  }
  CK(cudaStreamWaitEvent(sP, ev(count - 1, J.lookahead == 0 ? 0 : 1), 0));
  // results: this rank's L\U columns back into the host matrix, pivots from rank 0
  {
    int64_t cl = 0;
    for (int64_t j = r; j < count; j += P) {
      const int64_t w = std::min(b, n - j * b);
      CK(cudaMemcpy2DAsync(J.a + j * b, J.lda * 8, R.a + cl, ld * 8, w * 8, n, cudaMemcpyDeviceToHost, sP));
      cl += w;
    }
  }
  if (r == 0) CK(cudaMemcpyAsync(J.ipiv, R.piv, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, sP));
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, R.info, 8, cudaMemcpyDeviceToHost, sP));
  CK(cudaStreamSynchronize(sP));
  CK(cudaStreamSynchronize(sU));
  J.info[r] = h == ~0ull ? 0 : (int64_t)h;
  if (tracing) {
    int nrec = 0;
    for (const TRec& t : trecs) {
      if (nrec >= J.trace_cap) break;
      float s = 0.f, e = 0.f;
      CK(cudaEventElapsedTime(&s, t0, t.e0));
      CK(cudaEventElapsedTime(&e, t0, t.e1));
      J.trace[nrec++] = pflu_trace_event{t.label, t.k, s, e, 0.0};
    }
    J.trace_len = nrec;
  }
  return PFLU_OK;
}

static int mg_getrf(double* a, int64_t n, int64_t lda, int64_t b, int lookahead, int P, int64_t* ipiv,
                    int64_t* info, const pflu_options& opt, pflu_trace_event* trace, int trace_cap, int* trace_len) {
  if (g_mg.P != P) CKR(mg_init(P, nullptr));
  MgJob J{a, n, lda, b, lookahead, opt, ipiv, std::vector<int64_t>(P, 0), std::vector<int>(P, PFLU_OK),
          std::vector<std::string>(P), trace, trace_cap, 0};
  for (auto& R : g_mg.ranks) {
    R->packed.store(-1);
    R->received.store(-1);
  }
  // (pinned host memory gives every rank's strided copies full bandwidth; pageable memory works)
  std::vector<std::thread> th;
  for (int r = 0; r < P; ++r)
    th.emplace_back([&, r]() {
      J.rc[r] = mg_rank_run(*g_mg.ranks[r], J);
      if (J.rc[r] != PFLU_OK) J.err[r] = g_err;
    });
  for (auto& t : th) t.join();
  for (int r = 0; r < P; ++r)
    if (J.rc[r] != PFLU_OK) {
      g_err = "rank " + std::to_string(r) + ": " + J.err[r];
      return J.rc[r];
    }
  int64_t inf = 0;
  for (int64_t v : J.info)
    if (v > 0 && (inf == 0 || v < inf)) inf = v;
  if (info) *info = inf;
  if (trace_len) *trace_len = J.trace_len;
  return PFLU_OK;
}

}  // namespace pflu
