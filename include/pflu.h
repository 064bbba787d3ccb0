/*
 * pflu.h -- C ABI of libpflu.so, the B200 (sm_100a) LU-with-partial-pivoting library.
 *
 * Drop-in boundary for the reference package `panelforge` (arXiv 1804.07017), hot path
 * Kind.LU of dmf_la / dmf_mtb.  Plain C types only (no torch types); every function returns
 * PFLU_OK (0), a NEGATIVE value -i when argument i is invalid (LAPACK convention, 1-based),
 * or a POSITIVE PFLU_ERR_* code with a message in pflu_last_error().
 *
 * Conventions (all entry points):
 *   - matrices are float64 and ROW-MAJOR: element (i, j) at a[i * lda + j];
 *   - pivots are int64, 0-based, LAPACK ipiv semantics: for k ascending, row k was swapped with
 *     row ipiv[k] (ipiv[k] >= k).  The reference's LuOutput.pivots are these values + 1
 *     (pkg/src/panelforge/factor.py:51-62, 144);
 *   - `info` is 0, or 1 + the first column whose pivot was exactly zero; that column is left
 *     unscaled and the factorization completes (reference factor.py:56-58, _jit.py:171-174).
 *
 * Reference interfaces replaced (pkg/src/panelforge/...):
 *   pflu_getrf / pflu_getrf_device  <- dmf_la (factor.py:455-515, lookahead=1) and
 *                                      dmf_mtb (factor.py:382-412, lookahead=0), kind=Kind.LU
 *   pflu_panel                      <- _factor_panel + lu_unb + _jit.lu_unb_run
 *                                      (factor.py:128-144, 235-250; _jit.py:154-187)
 *   pflu_laswp                      <- laswp + _jit.laswp_run (kernels.py:273-300; _jit.py:141-151)
 *   pflu_swap_trsm                  <- _panel_laswp + trsm_llnu inside _update_columns
 *                                      (factor.py:253-277; kernels.py:225-246; _jit.py:104-113)
 *   pflu_trsm                       <- trsm_llnu (kernels.py:225-246; _jit.py:104-113)
 *   pflu_gemm_update                <- the gemm(A22, A21, -A12) of _update_columns
 *                                      (factor.py:278-285; kernels.py:173-218; _jit.py:54-80)
 *   pflu_init / pflu_getrf_mg /     <- the same dmf_la / dmf_mtb call on every GPU of the node
 *   pflu_finalize                      (optional init/finalize holding the comms)
 */
#ifndef PFLU_H
#define PFLU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFLU_OK 0
#define PFLU_ERR_CUDA 1        /* CUDA runtime/driver failure (see pflu_last_error) */
#define PFLU_ERR_NOMEM 2       /* device or pinned-host allocation failed */
#define PFLU_ERR_UNSUPPORTED 3 /* valid request this build cannot run (e.g. no sm_100 device) */

typedef struct pflu_options {
  int exact;        /* 1: every update in the reference's rounding (multiply, round, subtract):
                       results are bitwise equal to the reference; 0: trailing GEMM on DMMA */
  int panel_ctas;   /* CTAs of the panel kernel (0 = automatic; at most 16 for the cluster kernel) */
  int leaf_width;   /* leaf columns: 8, 16 or 32 (0 = automatic) */
  int panel_kernel; /* 0 automatic, 1 cooperative grid (LL exchange through L2), 2 one thread-block
                       cluster (DSMEM exchange; PFLU_ERR_UNSUPPORTED if the panel does not fit),
                       3 recursive: halves split down to 32-column leaves (persistent kernel), the
                       halves joined by swap+TRSM and a full-height DMMA GEMM,
                       4 several 16-CTA clusters (DSMEM exchange inside a cluster, one LL round through L2
                       between the clusters per column); panels under 8192 rows fall back to 1 */
  int malleable;    /* look-ahead 1 trailing update (the reference's LA / LA_MB, runtime.py:99-113):
                       0 dynamic: one CTA per GEMM tile, the block scheduler hands the panel's SMs
                         back to pending tiles as soon as the panel kernel exits (default);
                       1 LA: SM-partitioned -- a persistent GEMM on every SM but the ones the panel
                         kernel occupies (recorded from PF(0)); those stay with the panel chain;
                       2 LA_MB: as 1, and after PF(k+1) a join grid on the panel's SMs takes tiles of
                         TU_R(k) from the same atomic tile queue (the panel worker rejoining the team) */
  int reserved[3];
} pflu_options;

/* Trace record, one per timed task (labels as the reference's TraceEvent, factor.py:104-122). */
#define PFLU_TRACE_PF 0   /* panel factorization of step k             */
#define PFLU_TRACE_TU 1   /* full trailing update (lookahead 0)          */
#define PFLU_TRACE_TU_L 2 /* update of panel k+1's columns (lookahead 1) */
#define PFLU_TRACE_TU_R 3 /* remaining trailing update (lookahead 1)     */
#define PFLU_TRACE_GEMM 4 /* the DMMA GEMM inside TU / TU_R (roofline)   */
#define PFLU_TRACE_BCAST 5 /* multi-GPU: receipt of step k's panel + pivots (pflu_getrf_mg) */
typedef struct pflu_trace_event {
  int32_t label;
  int32_t k;
  float start_ms; /* CUDA-event time relative to the start of the factorization */
  float end_ms;
  double flop;    /* algorithmic flops of the traced work (GEMM records; 0 otherwise) */
} pflu_trace_event;

int pflu_version(void);
/* Cumulative number of kernels this library has launched in the process (bench evidence). */
long long pflu_launch_count(void);
/* Which record kinds a trace collects: bit (1 << PFLU_TRACE_x) per kind, default all.  Every record costs
   two event records on its stream (~2 us of GPU time each): a timed run that only needs the GEMM and PF
   records (bench.py's roofline) masks the rest.  Returns the previous mask. */
unsigned pflu_set_trace_mask(unsigned mask);
const char* pflu_last_error(void);
void pflu_default_options(pflu_options* opt);
int pflu_device_count(void);

/* Whole factorization, HOST buffers: stages H2D, factors, and streams every block row back as
 * soon as it is final (the D2H overlaps the rest of the factorization); pivots follow the last step.
 * a: m x n row-major (m >= n >= 1, lda >= n), overwritten with L\U in place; pinned memory gives
 * full PCIe bandwidth.  ipiv: int64[n] host.  lookahead: 0 (dmf_mtb order) or 1 (dmf_la).
 * The device copy is a grow-only workspace kept for the next call (see pflu_release_workspace). */
int pflu_getrf(double* a, int64_t m, int64_t n, int64_t lda, int64_t b, int lookahead,
               int64_t* ipiv, int64_t* info, const pflu_options* opt);

/* ---------------------------------------------------------------------------------------------
 * Multi-GPU: one process, P devices, one host thread per rank.
 * Reference interface replaced: the in-process dmf_la / dmf_mtb call (factor.py:455-456, 382-383)
 * reaching every GPU of the node.  1-D block-cyclic columns (block j on rank j % P), per step ONE
 * message (the owner's factored (n - kb) x b panel + its pivots) sent with ncclBroadcast over
 * NVLink (communicators from ncclCommInitAll; NCCL is dlopen'ed, not linked), look-ahead 1 across
 * ranks.  Ranks that share a device (tests on one GPU) exchange by device-to-device copies. */

/* Create (or re-create) the P-rank context: ranks on devices[0 .. P) (NULL: devices 0 .. P-1; a
 * device may repeat -- then the copy transport is used).  Holds the NCCL communicators, per-rank
 * streams and grow-only workspaces until pflu_finalize. */
int pflu_init(int n_gpus, const int* devices);
/* Destroy the communicators and free every rank's workspace. */
int pflu_finalize(void);
/* Ranks of the current multi-GPU context (0 if none); 1 if it uses NCCL, 0 for the copy transport. */
int pflu_mg_size(void);
int pflu_mg_uses_nccl(void);
/* Block-cyclic bookkeeping (host only): columns rank r of P stores for an n x n matrix, block b. */
int64_t pflu_mg_local_cols(int64_t n, int64_t b, int n_gpus, int rank);

/* Whole factorization of a square HOST matrix (n x n row-major, lda >= n, overwritten with L\U) on
 * n_gpus ranks; ipiv int64[n] host.  n_gpus == 1 is pflu_getrf (unless PFLU_MG_FORCE=1); n_gpus > 1
 * uses the current pflu_init context when it has n_gpus ranks, else creates one on devices
 * 0 .. n_gpus-1.  trace (optional): rank 0's PF / TU_L / TU_R (TU at look-ahead 0) / BCAST records. */
int pflu_getrf_mg(double* a, int64_t n, int64_t lda, int64_t b, int lookahead, int n_gpus, int64_t* ipiv,
                  int64_t* info, const pflu_options* opt, pflu_trace_event* trace, int trace_cap, int* trace_len);

/* Frees pflu_getrf's device workspace (synchronizes the device). */
int pflu_release_workspace(void);

/* Whole factorization, DEVICE buffers on the current device, ordered on `stream`
 * (a cudaStream_t; NULL = legacy default).  d_ipiv: int64[n] device.  Blocks until done and
 * writes *info on the host.  trace (optional, may be NULL) receives up to trace_cap events;
 * *trace_len (optional) the number written. */
int pflu_getrf_device(double* d_a, int64_t m, int64_t n, int64_t lda, int64_t b, int lookahead,
                      int64_t* d_ipiv, int64_t* info, void* stream, const pflu_options* opt,
                      pflu_trace_event* trace, int trace_cap, int* trace_len);

/* Panel factorization (getf2 semantics, recursive + cooperative leaf): rows [d, m) of the
 * w columns starting at column `col`; the diagonal of panel column j is row d + j.  Row
 * interchanges are applied across the panel's w columns only.  Writes d_ipiv[d .. d+min(w,m-d))
 * (global 0-based rows).  *info: 0 or 1 + first zero-pivot ROW index d + j.  With info == NULL the
 * call is asynchronous on `stream` (see pflu_info_reset / pflu_info_read). */
int pflu_panel(double* d_a, int64_t lda, int64_t m, int64_t d, int64_t col, int64_t w,
               int64_t* d_ipiv, int64_t* info, void* stream, const pflu_options* opt);

/* Strided 2-D copy (bytes; host or device pointers, unified addressing): `height` rows of `width`
 * bytes.  Moves a rank's block-cyclic columns between a host matrix and its device buffer. */
int pflu_copy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t height,
                void* stream);

/* Asynchronous info handling for pflu_panel(..., info = NULL, ...): reset / read (blocking) the
 * device-side "first zero pivot" word that asynchronous panel calls accumulate into. */
int pflu_info_reset(void* stream);
int pflu_info_read(int64_t* info, void* stream);

/* Compose the ascending swaps d_ipiv[d .. d+nb) into a gather plan (device int64[1 + 3*nb], caller
 * owned), for pflu_swap_trsm_plan.  Asynchronous on `stream`. */
int pflu_pivot_plan(const int64_t* d_ipiv, int64_t d, int64_t nb, int64_t* d_plan, void* stream);

/* laswp by a precomputed plan on columns [c0, c1) of rows >= d, then (if d_l != NULL) the nb top rows
 * (d .. d+nb) of those columns := unit_lower(L)^-1 * rows, L = d_l (nb x nb, leading dimension ldl).
 * Asynchronous; the multi-GPU driver's TU step for columns whose L11 lives in a broadcast buffer. */
int pflu_swap_trsm_plan(double* d_a, int64_t lda, int64_t d, int64_t nb, const int64_t* d_plan, int64_t c0,
                        int64_t c1, const double* d_l, int64_t ldl, void* stream);

/* Fast-mode solve support (not in the reference's rounding): d_inv (device, ceil(nb/32) * 1024
 * doubles) := the inverted 32x32 diagonal blocks of unit_lower(L), L = d_l (nb x nb, ld ldl). */
int pflu_diag_inv(const double* d_l, int64_t ldl, int64_t nb, double* d_inv, void* stream);

/* pflu_swap_trsm_plan with the solve on the DMMA tensor cores, using d_inv from pflu_diag_inv
 * (nb <= 512; larger nb falls back to the substitution of pflu_swap_trsm_plan). */
int pflu_swap_trsm_inv(double* d_a, int64_t lda, int64_t d, int64_t nb, const int64_t* d_plan, int64_t c0,
                       int64_t c1, const double* d_l, int64_t ldl, const double* d_inv, void* stream);

/* Row interchanges: for k = k1 .. k2-1 ascending, swap rows k and d_ipiv[k] on columns [c0, c1). */
int pflu_laswp(double* d_a, int64_t lda, int64_t c0, int64_t c1, const int64_t* d_ipiv, int64_t k1,
               int64_t k2, void* stream);

/* Fused: laswp of rows d_ipiv[d .. d+nb) on columns [c0, c1), then the nb top rows of those
 * columns := unit_lower(L11)^-1 * (rows), L11 = the nb x nb block at (d, lcol) of the same matrix. */
int pflu_swap_trsm(double* d_a, int64_t lda, int64_t d, int64_t lcol, int64_t nb, const int64_t* d_ipiv,
                   int64_t c0, int64_t c1, void* stream);

/* X (nb x ncols) := unit_lower(L)^-1 * X (strictly-upper part and diagonal of L ignored). */
int pflu_trsm(const double* d_l, int64_t ldl, int64_t nb, double* d_x, int64_t ldx, int64_t ncols,
              void* stream);

/* C (m x n) -= A (m x k) * B (k x n).  exact=1: reference rounding; exact=0: DMMA tensor cores. */
int pflu_gemm_update(double* d_c, int64_t ldc, const double* d_a, int64_t lda, const double* d_b,
                     int64_t ldb, int64_t m, int64_t n, int64_t k, int exact, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Householder QR (Kind.QR of dmf_mtb / dmf_la).  Same row-major storage;
 * the factors overwrite a in place: R on and above the diagonal, the Householder vectors' tails
 * below it (unit heads implicit), tau[j] the scalar of reflector j (H_j = I - tau_j v_j v_j^T;
 * tau_j = 0 is a null reflector for a column that is already zero below the diagonal).
 * Reference interfaces replaced (pkg/src/panelforge/...):
 *   pflu_geqrf / pflu_geqrf_device  <- dmf_mtb (factor.py:382-412, lookahead=0) and dmf_la
 *                                      (factor.py:455-515, lookahead=1) with kind=Kind.QR,
 *                                      returning QrOutput (factor.py:65-72)
 *   pflu_qr_panel                   <- qr_unb + _jit.qr_unb_run (factor.py:147-161; _jit.py:190-218)
 *   pflu_larft                      <- larft_forward_columnwise (factor.py:174-189)
 *   pflu_apply_block_reflector      <- apply_block_reflector (factor.py:192-205)
 * Block sizes up to 1024.  Results agree with the reference to rounding (the reference's own T is
 * formed with numpy/BLAS products), not bitwise. */

/* Whole factorization, HOST buffers (H2D, factorization, D2H).  a: m x n row-major (m >= n >= 1,
 * lda >= n), overwritten in place; tau: double[n] host. */
int pflu_geqrf(double* a, int64_t m, int64_t n, int64_t lda, int64_t b, int lookahead, double* tau);

/* Whole factorization, DEVICE buffers on the current device, ordered on `stream`; blocks until done.
 * d_tau: double[n] device.  trace (optional, may be NULL): PF / TU (look-ahead 0) or PF / TU_L / TU_R
 * records as for pflu_getrf_device (the reference's TraceEvent labels, factor.py:104-122). */
int pflu_geqrf_device(double* d_a, int64_t m, int64_t n, int64_t lda, int64_t b, int lookahead, double* d_tau,
                      void* stream, pflu_trace_event* trace, int trace_cap, int* trace_len);

/* Householder factorization of the panel rows [d, m) x columns [col, col + w) (the diagonal of
 * panel column j is row d + j; w <= m - d), in place; d_tau[0 .. w) receives the scalars.
 * Asynchronous on `stream`; one panel at a time per device (the leaf kernels' exchange buffers are
 * per device). */
int pflu_qr_panel(double* d_a, int64_t lda, int64_t m, int64_t d, int64_t col, int64_t w, double* d_tau,
                  void* stream);

/* T (k x k, upper, ld ldt, device) with H_1 ... H_k = I - V T V^T for the reflectors stored in the
 * mp x k panel d_v (ld ldv; unit diagonal implied, upper part ignored) and d_tau[0 .. k).  Blocks. */
int pflu_larft(const double* d_v, int64_t ldv, int64_t mp, int64_t k, const double* d_tau, double* d_t,
               int64_t ldt, void* stream);

/* C (mp x nc, ld ldc, device) := (H_1 ... H_k)^T C = C - V (T^T (V^T C)) for the reflectors stored in
 * the mp x k panel d_v with scalars d_tau.  Asynchronous on `stream`; workspaces are per stream, so
 * calls on different streams may run concurrently (the multi-GPU driver's TU_L / TU_R). */
int pflu_apply_block_reflector(const double* d_v, int64_t ldv, int64_t mp, int64_t k, const double* d_tau,
                               double* d_c, int64_t ldc, int64_t nc, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PFLU_H */
