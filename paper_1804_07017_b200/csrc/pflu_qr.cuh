// pflu_qr.cuh -- blocked Householder QR (Kind.QR) on the B200, SURVEY.md §8(f) row 4.
//
// Included by pflu.cu inside namespace pflu (after the GEMM launchers).  Same storage as the LU
// path: float64 m x n row-major, factored in place (R on/above the diagonal, the reflectors' tails
// below it, unit heads implicit), tau[n] out.  Reference (pkg/src/panelforge/...):
//   qr_leaf_kernel            <- qr_unb / _jit.qr_unb_run (factor.py:147-161, _jit.py:190-218),
//                                32 columns at a time
//   qr_larft_kernel           <- larft_forward_columnwise (factor.py:174-189)
//   qr_apply (3 DMMA GEMMs)   <- apply_block_reflector (factor.py:192-205): C - V (T^T (V^T C))
//   geqrf_async               <- dmf_mtb (factor.py:382-412, depth 0) / dmf_la (factor.py:455-515,
//                                depth 1) with kind=Kind.QR
//
// B200 mapping.  The panel (m_p x b) is factored in 32-column leaves by ONE cooperative kernel per
// leaf: every CTA keeps its contiguous row chunk of the leaf in shared memory for all 32 columns,
// and each column costs two grid-wide exchanges (the column norm's partial sums, then the partial
// dot products v^T a_c of the leaf's later columns), each reduced by every CTA in the same fixed
// order so all CTAs hold bit-identical tau / s_c.  Between leaves, and for the trailing matrix,
// the reflectors are applied as a block reflector on the FP64 tensor cores: V^T C and V^T V are
// tall-skinny products (K = panel height) run as split-K DMMA GEMMs whose slices are summed in a
// fixed order (deterministic), T^T W and C -= V Z are the ordinary DMMA GEMM.
#pragma once

namespace pflu {

constexpr int QR_THREADS = 256;
constexpr int QR_LW = 32;   // leaf width
constexpr int QR_LDT = 33;  // leaf tile row stride (doubles)
constexpr int QR_MAXG = 256;

static int g_qr_rows = []() { const char* e = getenv("PFLU_QR_ROWS"); return e ? atoi(e) : 256; }();  // 512: n=4096 QR 36.5 -> 31.8 ms at 256
static int g_qr_cluster = []() { const char* e = getenv("PFLU_QR_CLUSTER"); return e ? atoi(e) : 1; }();

struct QrLeafArgs {
  double* a;
  int64_t lda;
  int64_t r0, m;   // leaf rows [r0, m); the diagonal of leaf column j is row r0 + j
  int64_t c0;      // leaf columns [c0, c0 + w)
  int w;
  int G, R;        // CTAs, rows per CTA
  double* tau;     // tau of leaf column j at tau[j]
  double* dots;    // [2][G][32] partial x^T a_c (column parity)
  double* drow;    // [2][32] diagonal row
  double* gram;    // [G][32 x 32] partial V^T V of the finished leaf
  unsigned* bar;   // grid barrier counter, zeroed before the launch
  // the enclosing panel's block reflector (rows [r0 - p0, m)): this leaf writes its columns
  // [p0, p0 + w) of V (vd, ld ldv) and V^T (vt, ld ldvt), zeros above, and its diagonal block of
  // T^T (tt, ld ldt)
  double* vd;
  int64_t ldv;
  double* vt;
  int64_t ldvt;
  double* tt;
  int64_t ldt;
  int p0;
};

__device__ __forceinline__ double qr_warp_sum(double v) {
  // xor butterfly: every lane ends with the bit-identical sum
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void qr_grid_sync(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// Sum of the G partials at src[0..G) (L2 reads), same order on every CTA.
__device__ __forceinline__ double qr_sum_partials(const double* src, int G, int stride, int lane) {
  double t = 0.0;
  for (int i = lane; i < G; i += 32) t += __ldcg(src + (int64_t)i * stride);
  return qr_warp_sum(t);
}

// One grid exchange per column: with x the column below the diagonal and v = x * scale, the
// reflector's products s_c = a_jc + v^T a_c equal a_jc + scale * (x^T a_c), so the squared norm
// (c = j) and every raw dot x^T a_c (c > j) are reduced together BEFORE the norm is known; every
// CTA then derives beta, tau, scale and s_c from the same sums (same order, same bits) and updates
// its rows.  Rounding differs from the reference's sequential order (parity is to tolerance).
// After the last column the leaf also emits its part of the panel's block reflector: V and V^T
// (unit diagonal, zeros above) and, from one more exchange of partial Gram matrices, its 32x32
// diagonal block of T (the column recurrence of larft, factor.py:174-189) -- so the in-panel block
// reflector needs no separate make-V / Gram / larft launches.
// (An NCCL-LL style variant without the grid barrier -- flagged 16-byte partials polled by every
// CTA -- measured slower: 0.264 vs 0.214 ms per 32768 x 32 leaf, polling contention on shared lines.)
//
// CL = true (panels of <= ~13500 rows): the CTAs form ONE thread-block cluster and the exchange goes
// through distributed shared memory -- every CTA stores its partials straight into each peer's
// shared memory and a cluster barrier (release/acquire) replaces the global grid barrier and the
// L2 round trip of the reads.
constexpr int QR_CL_MAX = 16;
template <bool CL>
__global__ void __launch_bounds__(QR_THREADS, 1) qr_leaf_kernel(QrLeafArgs p) {
  extern __shared__ __align__(16) double qr_smem[];
  double* tile = qr_smem;  // R x QR_LDT
  double* xs = qr_smem + p.R * QR_LDT;   // CL: [2][QR_CL_MAX][32] peers' partials
  double* xd = xs + 2 * QR_CL_MAX * QR_LW;  // CL: [2][32] diagonal row
  __shared__ double sc[QR_LW];   // column sums, then s_c
  __shared__ double dr[QR_LW];   // diagonal row
  __shared__ double tl[QR_LW];   // tau of the leaf's columns
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q = blockIdx.x;
  constexpr int NW = QR_THREADS / 32;
  const int64_t rbeg = p.r0 + (int64_t)q * p.R;
  const int64_t rend = min(p.m, rbeg + p.R);
  const int nrows = (int)max((int64_t)0, rend - rbeg);
  const int w = p.w;
  for (int idx = tid; idx < nrows * w; idx += QR_THREADS) {
    const int r = idx / w, c = idx - r * w;
    tile[r * QR_LDT + c] = p.a[(rbeg + r) * p.lda + p.c0 + c];
  }
  if constexpr (CL) cl_sync();  // every peer is running before the first DSMEM store
  else __syncthreads();
  for (int j = 0; j < w; ++j) {
    const int64_t d = p.r0 + j;
    const int par = j & 1;
    const bool own_d = d >= rbeg && d < rend;
    const int dl = (int)(d - rbeg);
    const int rfirst = (int)min((int64_t)nrows, max((int64_t)0, d + 1 - rbeg));
    double* dots = p.dots + (int64_t)par * p.G * QR_LW;
    // (A) partial x^T a_c for c in [j, w) over this CTA's rows below the diagonal, one warp per column
    for (int c = j + warp; c < w; c += NW) {
      double t = 0.0, t1 = 0.0;
      int r = rfirst + lane;
      for (; r + 32 < nrows; r += 64) {
        t += tile[r * QR_LDT + j] * tile[r * QR_LDT + c];
        t1 += tile[(r + 32) * QR_LDT + j] * tile[(r + 32) * QR_LDT + c];
      }
      if (r < nrows) t += tile[r * QR_LDT + j] * tile[r * QR_LDT + c];
      t = qr_warp_sum(t + t1);
      if constexpr (CL) {
        if (lane < p.G) {
          const uint32_t xa = smem_addr(xs + (par * QR_CL_MAX + q) * QR_LW + c);
          asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(cl_map(xa, lane)), "d"(t) : "memory");
          if (own_d) {
            const uint32_t da = smem_addr(xd + par * QR_LW + c);
            asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(cl_map(da, lane)), "d"(tile[dl * QR_LDT + c])
                         : "memory");
          }
        }
      } else if (lane == 0) {
        dots[(int64_t)q * QR_LW + c] = t;
        if (own_d) p.drow[par * 32 + c] = tile[dl * QR_LDT + c];
      }
    }
    if constexpr (CL) cl_sync();
    else qr_grid_sync(p.bar, (unsigned)(j + 1) * (unsigned)p.G);
    // (B) the same fixed-order sums on every CTA; all loads of a warp's columns in flight together
    {
      double acc[(QR_LW + NW - 1) / NW];
#pragma unroll
      for (int u = 0; u < (QR_LW + NW - 1) / NW; ++u) acc[u] = 0.0;
      if constexpr (CL) {
        if (lane < p.G) {
#pragma unroll
          for (int u = 0; u < (QR_LW + NW - 1) / NW; ++u) {
            const int c = j + warp + u * NW;
            if (c < w) acc[u] = xs[(par * QR_CL_MAX + lane) * QR_LW + c];
          }
        }
      } else {
        // every load of the warp's columns issued before the first add (G <= QR_MAXG)
        double v[QR_MAXG / 32][(QR_LW + NW - 1) / NW];
#pragma unroll
        for (int t = 0; t < QR_MAXG / 32; ++t)
#pragma unroll
          for (int u = 0; u < (QR_LW + NW - 1) / NW; ++u) {
            const int i = lane + 32 * t, c = j + warp + u * NW;
            v[t][u] = (i < p.G && c < w) ? __ldcg(dots + (int64_t)i * QR_LW + c) : 0.0;
          }
#pragma unroll
        for (int t = 0; t < QR_MAXG / 32; ++t)
#pragma unroll
          for (int u = 0; u < (QR_LW + NW - 1) / NW; ++u) acc[u] += v[t][u];
      }
#pragma unroll
      for (int u = 0; u < (QR_LW + NW - 1) / NW; ++u) {
        const int c = j + warp + u * NW;
        const double t = qr_warp_sum(acc[u]);
        if (lane == 0 && c < w) {
          sc[c] = t;
          dr[c] = CL ? xd[par * QR_LW + c] : __ldcg(p.drow + par * 32 + c);
        }
      }
    }
    __syncthreads();
    const double sq = sc[j], alpha = dr[j];
    if (sq == 0.0) {  // null reflector, column unchanged (uniform over the grid; _jit.py:203-205)
      if (tid == 0) {
        tl[j] = 0.0;
        if (q == 0) p.tau[j] = 0.0;
      }
      __syncthreads();
      continue;
    }
    const double norm = sqrt(alpha * alpha + sq);
    const double beta = alpha >= 0.0 ? -norm : norm;
    const double tj = (beta - alpha) / beta;
    const double scale = 1.0 / (alpha - beta);
    if (tid == 0) {
      tl[j] = tj;
      if (q == 0) p.tau[j] = tj;
    }
    __syncthreads();  // every thread read sc[j] before it is overwritten below
    if (tid < w && tid > j) sc[tid] = (dr[tid] + scale * sc[tid]) * tj;
    __syncthreads();
    // (C) v = x * scale; a_ic -= s_c v_i; a_jj = beta; a_jc -= s_c (_jit.py:206-218)
    for (int r = rfirst + tid; r < nrows; r += QR_THREADS) {
      double* tr = tile + r * QR_LDT;
      const double v = tr[j] * scale;
      tr[j] = v;
      for (int c = j + 1; c < w; ++c) tr[c] -= sc[c] * v;
    }
    if (own_d) {
      if (tid == 0) tile[dl * QR_LDT + j] = beta;
      for (int c = j + 1 + tid; c < w; c += QR_THREADS) tile[dl * QR_LDT + c] -= sc[c];
    }
    __syncthreads();
  }
  // write back; V (row-major) and V^T of the leaf's columns into the panel's reflector block
  const int64_t rho0 = rbeg - p.r0;  // leaf-local index of this CTA's first row
  auto vval = [&](int r, int c) -> double {
    const int64_t rho = rho0 + r;
    return rho > c ? tile[r * QR_LDT + c] : (rho == c ? 1.0 : 0.0);
  };
  for (int idx = tid; idx < nrows * w; idx += QR_THREADS) {
    const int r = idx / w, c = idx - r * w;
    p.a[(rbeg + r) * p.lda + p.c0 + c] = tile[r * QR_LDT + c];
    p.vd[(p.p0 + rho0 + r) * p.ldv + p.p0 + c] = vval(r, c);
  }
  for (int idx = tid; idx < nrows * w; idx += QR_THREADS) {
    const int c = idx / nrows, r = idx - c * nrows;
    p.vt[(int64_t)(p.p0 + c) * p.ldvt + p.p0 + rho0 + r] = vval(r, c);
  }
  if (q == 0) {  // rows of the panel above this leaf: zeros in the leaf's columns
    for (int idx = tid; idx < p.p0 * w; idx += QR_THREADS) {
      const int r = idx / w, c = idx - r * w;
      p.vd[(int64_t)r * p.ldv + p.p0 + c] = 0.0;
    }
    for (int idx = tid; idx < p.p0 * w; idx += QR_THREADS) {
      const int c = idx / p.p0, r = idx - c * p.p0;
      p.vt[(int64_t)(p.p0 + c) * p.ldvt + r] = 0.0;
    }
  }
  // partial Gram v_x^T v_y (x < y) over this CTA's rows: rows below y contribute v_rx v_ry, row y v_yx
  for (int e = tid; e < w * w; e += QR_THREADS) {
    const int x = e / w, y = e - x * w;
    if (x >= y) continue;
    double acc = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // four chains: latency, not throughput, bound
    const int rs = (int)min((int64_t)nrows, max((int64_t)0, y - rho0));
    if (rs < nrows && rho0 + rs == y) acc = tile[rs * QR_LDT + x];
    int r = (rho0 + rs == y && rs < nrows) ? rs + 1 : rs;
    for (; r + 3 < nrows; r += 4) {
      acc += tile[r * QR_LDT + x] * tile[r * QR_LDT + y];
      a1 += tile[(r + 1) * QR_LDT + x] * tile[(r + 1) * QR_LDT + y];
      a2 += tile[(r + 2) * QR_LDT + x] * tile[(r + 2) * QR_LDT + y];
      a3 += tile[(r + 3) * QR_LDT + x] * tile[(r + 3) * QR_LDT + y];
    }
    for (; r < nrows; ++r) acc += tile[r * QR_LDT + x] * tile[r * QR_LDT + y];
    p.gram[(int64_t)q * QR_LW * QR_LW + x * QR_LW + y] = (acc + a1) + (a2 + a3);
  }
  if constexpr (CL) cl_sync();  // release/acquire at cluster scope covers the global partials
  else qr_grid_sync(p.bar, (unsigned)(w + 1) * (unsigned)p.G);
  if (q != 0) return;
  // CTA 0: G = sum of the partials (fixed order), T by the column recurrence, T^T block out
  double* gs = qr_smem;                  // 32 x 33 (the tile is no longer needed)
  double* ts = qr_smem + QR_LW * QR_LDT; // 32 x 33
  for (int e = tid; e < w * w; e += QR_THREADS) {
    const int x = e / w, y = e - x * w;
    double acc = 0.0;
    if (x < y)
      for (int i = 0; i < p.G; ++i) acc += __ldcg(p.gram + (int64_t)i * QR_LW * QR_LW + x * QR_LW + y);
    gs[x * QR_LDT + y] = acc;
    ts[x * QR_LDT + y] = 0.0;
  }
  __syncthreads();
  if (warp == 0) {
    const int i = lane;
    for (int j = 0; j < w; ++j) {
      double acc = 0.0;
      if (i < j)
        for (int l = i; l < j; ++l) acc += ts[i * QR_LDT + l] * gs[l * QR_LDT + j];
      __syncwarp();
      if (i < j) ts[i * QR_LDT + j] = -tl[j] * acc;
      else if (i == j) ts[i * QR_LDT + j] = tl[j];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < w * w; e += QR_THREADS) {
    const int r = e / w, c = e - r * w;  // tt[r][c] = T[c][r]
    p.tt[(int64_t)(p.p0 + r) * p.ldt + p.p0 + c] = c <= r ? ts[c * QR_LDT + r] : 0.0;
  }
}

// Dense reflector block of the panel rows [d, d + mp), columns [cv, cv + k): unit diagonal, zeros
// above.  vd: mp x k (ld ldv), vt = vd^T: k x mp (ld ldvt).  32x32 tiles through shared memory.
__global__ void qr_make_v_kernel(const double* __restrict__ a, int64_t lda, int64_t d, int64_t cv, int64_t mp,
                                 int k, double* __restrict__ vd, int64_t ldv, double* __restrict__ vt,
                                 int64_t ldvt) {
  __shared__ double t[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = i0 + r;
    const int c = c0 + tx;
    double v = 0.0;
    if (i < mp && c < k) v = i > c ? a[(d + i) * lda + cv + c] : (i == c ? 1.0 : 0.0);
    t[r][tx] = v;
    if (i < mp && c < k) vd[i * ldv + c] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int c = c0 + r;
    const int64_t i = i0 + tx;
    if (c < k && i < mp) vt[(int64_t)c * ldvt + i] = t[tx][r];
  }
}

// out (rows x cols, ld ldo) = sum over s of part[s] (slices cslice apart, ld ldp), s ascending.
__global__ void qr_split_reduce_kernel(const double* __restrict__ part, int64_t ldp, int64_t cslice, int S,
                                       int64_t rows, int64_t cols, double* __restrict__ out, int64_t ldo) {
  const int64_t n = rows * cols;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols, c = idx - r * cols;
    const double* src = part + r * ldp + c;
    double acc = src[0];
    for (int s = 1; s < S; ++s) acc += src[(int64_t)s * cslice];
    out[r * ldo + c] = acc;
  }
}

// larft (factor.py:174-189): T[j][j] = tau_j, T[:j, j] = -tau_j T[:j, :j] (V^T v_j), from
// gneg = -(V^T V).  Writes tt = T^T (k x k, ld ldt) including the zero upper part.
// Blocked over 32-column blocks (one CTA of 1024 threads, k <= 512): every diagonal block by its own
// warp with the column recurrence, then block column J from the merge rule of two compact-WY
// factors, T[0:J0, J] = -T[0:J0, 0:J0] (G[0:J0, J] T_JJ) -- the same T, rounded differently.
constexpr int QR_LARFT_THREADS = 1024;
constexpr int QR_LARFT_MAXK = 512;
__global__ void __launch_bounds__(QR_LARFT_THREADS, 1)
qr_larft_kernel(const double* __restrict__ gneg, int64_t ldg, const double* __restrict__ tau, int k, double* tt,
                int64_t ldt, int diag_given) {
  extern __shared__ double qr_x[];  // (QR_LARFT_MAXK - 32) x 32: G[0:J0, J] T_JJ, then T_JJ (32 x 33)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t idx = tid; idx < (int64_t)k * k; idx += QR_LARFT_THREADS) {
    const int r = (int)(idx / k), c = (int)(idx - (int64_t)r * k);
    if (c > r && (!diag_given || (c >> 5) != (r >> 5))) tt[(int64_t)r * ldt + c] = 0.0;  // given diagonal blocks stay
  }
  const int nb = (k + 31) / 32;
  // diagonal blocks (unless the leaf kernels already wrote them): lane i owns row i of T_II;
  // T[i][l] lives at tt[l][i]
  for (int bI = diag_given ? nb : warp; bI < nb; bI += QR_LARFT_THREADS / 32) {
    const int I0 = bI * 32, bs = min(32, k - I0);
    for (int j = 0; j < bs; ++j) {
      const double tj = tau[I0 + j];
      const int i = lane;
      double acc = 0.0;
      if (i < j)
        for (int l = i; l < j; ++l) acc += tt[(int64_t)(I0 + l) * ldt + I0 + i] * -gneg[(int64_t)(I0 + l) * ldg + I0 + j];
      __syncwarp();
      if (i < j) tt[(int64_t)(I0 + j) * ldt + I0 + i] = -tj * acc;
      else if (i == j) tt[(int64_t)(I0 + j) * ldt + I0 + j] = tj;
      __syncwarp();
    }
  }
  __syncthreads();
  // block column J: warp w owns rows r = w, w + 32, ...; lane = column c of the block
  double* tjj = qr_x + (size_t)(QR_LARFT_MAXK - 32) * 32;  // 32 x 33: T_JJ
  for (int bJ = 1; bJ < nb; ++bJ) {
    const int J0 = bJ * 32, bs = min(32, k - J0);
    for (int e = tid; e < 32 * 32; e += QR_LARFT_THREADS) {
      const int l = e >> 5, c = e & 31;  // T_JJ[l][c] = tt[J0 + c][J0 + l]
      tjj[l * 33 + c] = (l < bs && c < bs) ? tt[(int64_t)(J0 + c) * ldt + J0 + l] : 0.0;
    }
    __syncthreads();
    // X[r][c] = sum_{l <= c} G[r][J0 + l] T_JJ[l][c]: the warp's G rows prefetched, then shuffles
    {
      double g[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int r = warp + 32 * t;
        g[t] = (r < J0 && lane < bs) ? -gneg[(int64_t)r * ldg + J0 + lane] : 0.0;
      }
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int r = warp + 32 * t;
        if (r >= J0) break;
        double acc = 0.0;
        for (int l = 0; l < 32; ++l) {
          const double gl = __shfl_sync(0xffffffffu, g[t], l);
          if (l <= lane) acc += gl * tjj[l * 33 + lane];
        }
        qr_x[r * 32 + lane] = acc;
      }
    }
    __syncthreads();
    // T[r][J0 + c] = -sum_{l = r}^{J0 - 1} T[r][l] X[l][c]; T[r][l] = tt[l][r], 32 l per load round
    for (int r = warp; r < J0; r += QR_LARFT_THREADS / 32) {
      double tv[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int l = r + 32 * t + lane;
        tv[t] = l < J0 ? tt[(int64_t)l * ldt + r] : 0.0;
      }
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int l0 = r + 32 * t;
        if (l0 >= J0) break;
        const int cnt = min(32, J0 - l0);
        for (int i = 0; i < cnt; ++i) acc += __shfl_sync(0xffffffffu, tv[t], i) * qr_x[(l0 + i) * 32 + lane];
      }
      if (lane < bs) tt[(int64_t)(J0 + lane) * ldt + r] = -acc;
    }
    __syncthreads();
  }
}

// One block column J of T when the diagonal blocks are given (the factorization path): one launch
// per J, CTA b owns rows 8b .. 8b + 7 of T[0:J0, J]; every CTA forms the whole X = G[0:J0, J] T_JJ in
// shared memory (cheap) so the CTAs need no exchange.  Also zeroes tt's upper entries in block J.
constexpr int QR_MERGE_ROWS = 8;
__global__ void __launch_bounds__(QR_MERGE_ROWS * 32)
qr_larft_merge_kernel(const double* __restrict__ gneg, int64_t ldg, int k, int J0, double* tt, int64_t ldt) {
  extern __shared__ double qr_mx[];  // X: J0 x 32, then T_JJ: 32 x 33
  double* tjj = qr_mx + (size_t)J0 * 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bs = min(32, k - J0);
  for (int e = tid; e < 32 * 32; e += QR_MERGE_ROWS * 32) {
    const int l = e >> 5, c = e & 31;  // T_JJ[l][c] = tt[J0 + c][J0 + l]
    tjj[l * 33 + c] = (l < bs && c < bs) ? tt[(int64_t)(J0 + c) * ldt + J0 + l] : 0.0;
  }
  __syncthreads();
  for (int r = warp; r < J0; r += QR_MERGE_ROWS) {
    const double g = lane < bs ? -gneg[(int64_t)r * ldg + J0 + lane] : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      const double gl = __shfl_sync(0xffffffffu, g, l);
      if (l <= lane) acc += gl * tjj[l * 33 + lane];
    }
    qr_mx[r * 32 + lane] = acc;
  }
  __syncthreads();
  const int r = blockIdx.x * QR_MERGE_ROWS + warp;
  if (r >= J0) return;
  double acc = 0.0;
  for (int l0 = r; l0 < J0; l0 += 32) {
    const double tv = l0 + lane < J0 ? tt[(int64_t)(l0 + lane) * ldt + r] : 0.0;
    const int cnt = min(32, J0 - l0);
    for (int i = 0; i < cnt; ++i) acc += __shfl_sync(0xffffffffu, tv, i) * qr_mx[(l0 + i) * 32 + lane];
  }
  if (lane < bs) {
    tt[(int64_t)(J0 + lane) * ldt + r] = -acc;
    tt[(int64_t)r * ldt + J0 + lane] = 0.0;
  }
}

// Column recurrence in one CTA (any k <= 1024; used above QR_LARFT_MAXK).
__global__ void qr_larft_seq_kernel(const double* __restrict__ gneg, int64_t ldg, const double* __restrict__ tau,
                                    int k, double* tt, int64_t ldt) {
  extern __shared__ double qr_y[];
  for (int64_t idx = threadIdx.x; idx < (int64_t)k * k; idx += blockDim.x) {
    const int r = (int)(idx / k), c = (int)(idx - (int64_t)r * k);
    if (c > r) tt[(int64_t)r * ldt + c] = 0.0;
  }
  const int i = threadIdx.x;
  for (int j = 0; j < k; ++j) {
    if (i < j) qr_y[i] = -gneg[(int64_t)i * ldg + j];
    __syncthreads();
    const double tj = tau[j];
    if (i < j) {
      double acc = 0.0;
      for (int l = i; l < j; ++l) acc += tt[(int64_t)l * ldt + i] * qr_y[l];
      tt[(int64_t)j * ldt + i] = -tj * acc;
    } else if (i == j) {
      tt[(int64_t)j * ldt + j] = tj;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------
// host side

static inline int64_t qr_even(int64_t x) { return (x + 1) & ~(int64_t)1; }

struct QrBuf {
  double* p = nullptr;
  size_t cap = 0;  // doubles
  int need(size_t n) {
    if (n <= cap) return PFLU_OK;
    // growing frees the old buffer: queued kernels may still use it (geqrf_async reserves every
    // buffer at its maximum before its first launch, so this only happens between calls)
    if (p) CK(cudaDeviceSynchronize());
    if (p) CK(cudaFree(p));
    p = nullptr;
    cap = 0;
    if (cudaMalloc(&p, n * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return set_err(PFLU_ERR_NOMEM, "QR workspace: cudaMalloc(%zu bytes) failed", n * sizeof(double));
    }
    cap = n;
    return PFLU_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// One block reflector: dense V, V^T and T^T.
struct QrRefl {
  QrBuf vd, vt, tt;
  int64_t mp = 0, ldv = 0, ldvt = 0, ldt = 0;
  int k = 0;
};

// Scratch of one stream: products W / Z / Gram and split-K slices.
struct QrScratch {
  QrBuf w, z, g, part;
};

// Workspace of the kernel-level entry points on one stream (the multi-GPU driver applies block
// reflectors on two streams at once).
struct QrSlot {
  cudaStream_t st = nullptr;
  QrRefl refl;
  QrScratch ws;
};

struct QrCtx {
  QrRefl refl[2];     // outer step reflectors, by step parity
  QrRefl leaf;        // pflu_qr_panel's reflector block
  std::vector<QrSlot*> slots;  // pflu_larft / pflu_apply_block_reflector, one per stream
  QrScratch ws[2];    // 0: panel stream (leaves, TU_L), 1: trailing stream (TU_R)
  QrBuf htau;         // pflu_geqrf: device tau (grow-only)
  static constexpr int RING = 8;
  QrRefl ring[RING];            // pflu_geqrf's chunked schedule: reflectors of the last RING steps
  QrScratch wsc[8];             // ... and one scratch per trailing column-chunk stream
  double* leafx = nullptr;  // leaf kernel exchange: dots, drow, partial Gram matrices
  unsigned* bar = nullptr;
  bool ready = false;
  void release() {
    for (QrRefl* r : {&refl[0], &refl[1], &leaf}) { r->vd.release(); r->vt.release(); r->tt.release(); }
    for (auto& r : ring) { r.vd.release(); r.vt.release(); r.tt.release(); }
    for (auto& w : ws) { w.w.release(); w.z.release(); w.g.release(); w.part.release(); }
    for (auto& w : wsc) { w.w.release(); w.z.release(); w.g.release(); w.part.release(); }
    htau.release();
    for (QrSlot* sl : slots) {
      sl->refl.vd.release(); sl->refl.vt.release(); sl->refl.tt.release();
      sl->ws.w.release(); sl->ws.z.release(); sl->ws.g.release(); sl->ws.part.release();
      delete sl;
    }
    slots.clear();
  }
  QrSlot& slot(cudaStream_t st) {
    for (QrSlot* sl : slots)
      if (sl->st == st) return *sl;
    if (slots.size() >= 8) {  // callers that create fresh streams per call: recycle the oldest slot
      cudaDeviceSynchronize();
      QrSlot* old = slots.front();
      old->refl.vd.release(); old->refl.vt.release(); old->refl.tt.release();
      old->ws.w.release(); old->ws.z.release(); old->ws.g.release(); old->ws.part.release();
      delete old;
      slots.erase(slots.begin());
    }
    slots.push_back(new QrSlot());
    slots.back()->st = st;
    return *slots.back();
  }
};
static QrCtx g_qr[64];

static int qr_ctx(DevCtx& c, QrCtx** out) {
  QrCtx& q = g_qr[c.dev];
  if (!q.ready) {
    CK(cudaMalloc(&q.leafx, sizeof(double) * (2 * QR_MAXG * QR_LW + 64 + QR_MAXG * QR_LW * QR_LW)));
    CK(cudaMalloc(&q.bar, 64));
    CK(cudaFuncSetAttribute(qr_larft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(sizeof(double) * ((QR_LARFT_MAXK - 32) * 32 + 32 * 33))));
    CK(cudaFuncSetAttribute(qr_larft_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(sizeof(double) * ((QR_LARFT_MAXK - 32) * 32 + 32 * 33))));
    CK(cudaFuncSetAttribute(qr_leaf_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)std::min<size_t>(c.smem_optin, 227 * 1024) - 1024));
    CK(cudaFuncSetAttribute(qr_leaf_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)std::min<size_t>(c.smem_optin, 227 * 1024) - 1024));
    CK(cudaFuncSetAttribute(qr_leaf_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    q.ready = true;
  }
  *out = &q;
  return PFLU_OK;
}

// A block reflector as the GEMMs see it (possibly a sub-block of a QrRefl).
struct QrView {
  const double* vd;
  int64_t ldv;
  const double* vt;
  int64_t ldvt;
  const double* tt;
  int64_t ldt;
  int64_t mp;
  int k;
};
static QrView qr_view(const QrRefl& R) { return {R.vd.p, R.ldv, R.vt.p, R.ldvt, R.tt.p, R.ldt, R.mp, R.k}; }

static int qr_refl_alloc(QrRefl& R, int64_t mp, int k) {
  R.mp = mp;
  R.k = k;
  R.ldv = qr_even(k);
  R.ldvt = qr_even(mp);
  R.ldt = qr_even(k);
  CKR(R.vd.need((size_t)(R.mp * R.ldv)));
  CKR(R.vt.need((size_t)(k * R.ldvt)));
  CKR(R.tt.need((size_t)(k * R.ldt)));
  return PFLU_OK;
}

static int qr_larft_launch(QrScratch& ws, QrRefl& R, const double* d_tau, int diag_given, cudaStream_t st) {
  const int k = R.k;
  if (diag_given && k <= QR_LARFT_MAXK) {
    for (int J0 = 32; J0 < k; J0 += 32) {
      qr_larft_merge_kernel<<<(J0 + QR_MERGE_ROWS - 1) / QR_MERGE_ROWS, QR_MERGE_ROWS * 32,
                              sizeof(double) * ((size_t)J0 * 32 + 32 * 33), st>>>(ws.g.p, R.ldt, k, J0, R.tt.p, R.ldt);
      CK(cudaGetLastError());
      g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return PFLU_OK;
  }
  if (k <= QR_LARFT_MAXK) {
    qr_larft_kernel<<<1, QR_LARFT_THREADS, sizeof(double) * ((QR_LARFT_MAXK - 32) * 32 + 32 * 33), st>>>(
        ws.g.p, R.ldt, d_tau, k, R.tt.p, R.ldt, diag_given);
  } else {
    const int thr = std::max(32, (k + 31) / 32 * 32);
    if (thr > 1024) return set_err(PFLU_ERR_UNSUPPORTED, "QR block size %d > 1024", k);
    qr_larft_seq_kernel<<<1, thr, sizeof(double) * k, st>>>(ws.g.p, R.ldt, d_tau, k, R.tt.p, R.ldt);
  }
  CK(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return PFLU_OK;
}

// Split-K DMMA product: out (M x N, ld ldo) = -(A B), A: M x K (ld lda), B: K x N (ld ldb).
static int qr_gemm_neg(DevCtx& c, QrScratch& ws, double* out, int64_t ldo, const double* a, int64_t lda,
                       const double* b, int64_t ldb, int64_t M, int64_t N, int64_t K, cudaStream_t st) {
  using C = GV6;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(gemm_dmma_t<C, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    CK(cudaFuncSetAttribute(gemm_dmma_t<C, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  if (M <= 0 || N <= 0) return PFLU_OK;
  const int64_t tm = (M + C::BM - 1) / C::BM, tn = (N + C::BN - 1) / C::BN;
  if (tm * tn > INT_MAX) return set_err(PFLU_ERR_UNSUPPORTED, "gemm grid too large");
  const int64_t want = std::max<int64_t>(1, (2 * c.sms + tm * tn - 1) / (tm * tn));
  int64_t S = std::max<int64_t>(1, std::min<int64_t>(want, (K + 255) / 256));
  S = std::min<int64_t>(S, 65535);
  int64_t ks = ((K + S - 1) / S + C::BK - 1) / C::BK * C::BK;
  if (K <= 0) ks = 0;
  S = K <= 0 ? 1 : (K + ks - 1) / ks;
  GemmArgs p;
  p.a = a; p.b = b; p.lda = lda; p.ldb = ldb;
  p.M = M; p.N = N; p.K = std::max<int64_t>(K, 0);
  p.tiles_m = (int)tm; p.tiles_n = (int)tn;
  p.kslice = std::max<int64_t>(ks, 1);
  if (S == 1) {
    p.c = out; p.ldc = ldo; p.cslice = 0;
  } else {
    const int64_t ldp = qr_even(N);
    CKR(ws.part.need((size_t)(S * M * ldp)));
    p.c = ws.part.p; p.ldc = ldp; p.cslice = M * ldp;
  }
  const bool v2 = aligned16(p.c) && aligned16(a) && aligned16(b) && (p.ldc % 2 == 0) && (lda % 2 == 0) &&
                  (ldb % 2 == 0);
  dim3 grid((unsigned)(tm * tn), (unsigned)S);
  if (v2) gemm_dmma_t<C, 2, true><<<grid, C::THREADS, C::SMEM, st>>>(p);
  else gemm_dmma_t<C, 1, true><<<grid, C::THREADS, C::SMEM, st>>>(p);
  CK(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (S > 1) {
    const int64_t n = M * N;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * c.sms);
    qr_split_reduce_kernel<<<blocks, 256, 0, st>>>(p.c, p.ldc, p.cslice, (int)S, M, N, out, ldo);
    CK(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  return PFLU_OK;
}

// V, V^T and T^T of the reflectors stored at rows [d, m), columns [cv, cv + k) (kernel-level
// entry points; the factorization gets V / V^T / T's diagonal blocks from the leaf kernels).
static int qr_build(DevCtx& c, QrScratch& ws, QrRefl& R, const double* a, int64_t lda, int64_t d, int64_t m,
                    int64_t cv, int k, const double* d_tau, cudaStream_t st) {
  CKR(qr_refl_alloc(R, m - d, k));
  dim3 g((unsigned)((R.mp + 31) / 32), (unsigned)((k + 31) / 32));
  qr_make_v_kernel<<<g, dim3(32, 8), 0, st>>>(a, lda, d, cv, R.mp, k, R.vd.p, R.ldv, R.vt.p, R.ldvt);
  CK(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
  CKR(ws.g.need((size_t)(k * R.ldt)));
  CKR(qr_gemm_neg(c, ws, ws.g.p, R.ldt, R.vt.p, R.ldvt, R.vd.p, R.ldv, k, k, R.mp, st));
  return qr_larft_launch(ws, R, d_tau, 0, st);
}

// T of a panel whose leaves already wrote V, V^T and T's 32x32 diagonal blocks: the Gram matrix
// on the split-K DMMA GEMM, then only the off-diagonal merges of larft.
static int qr_finish_t(DevCtx& c, QrScratch& ws, QrRefl& R, const double* d_tau, cudaStream_t st) {
  if (R.k <= 32) return PFLU_OK;
  CKR(ws.g.need((size_t)(R.k * R.ldt)));
  CKR(qr_gemm_neg(c, ws, ws.g.p, R.ldt, R.vt.p, R.ldvt, R.vd.p, R.ldv, R.k, R.k, R.mp, st));
  return qr_larft_launch(ws, R, d_tau, R.k <= QR_LARFT_MAXK ? 1 : 0, st);
}

// C (rows [d, m) of columns [lo, lo + nc)) := C - V (T^T (V^T C))   (factor.py:192-205)
static int qr_apply(DevCtx& c, QrScratch& ws, const QrView& R, double* cp, int64_t ldc, int64_t nc, cudaStream_t st) {
  if (nc <= 0 || R.k <= 0 || R.mp <= 0) return PFLU_OK;
  const int64_t ldw = qr_even(nc);
  CKR(ws.w.need((size_t)(R.k * ldw)));
  CKR(ws.z.need((size_t)(R.k * ldw)));
  // W = -(V^T C), Z = -(T^T W) = T^T V^T C, C -= V Z
  CKR(qr_gemm_neg(c, ws, ws.w.p, ldw, R.vt, R.ldvt, cp, ldc, R.k, nc, R.mp, st));
  CKR(qr_gemm_neg(c, ws, ws.z.p, ldw, R.tt, R.ldt, ws.w.p, ldw, R.k, nc, R.k, st));
  CKR(launch_gemm(cp, ldc, R.vd, R.ldv, ws.z.p, ldw, R.mp, nc, R.k, false, st));
  return PFLU_OK;
}

// Householder factorization of the panel rows [d, m), columns [col, col + w): 32-column leaves,
// each followed by its block reflector on the panel's remaining columns.  On return R holds the
// panel's V, V^T and the 32x32 diagonal blocks of T^T (qr_finish_t completes T).
static int qr_panel(DevCtx& c, QrCtx& q, double* a, int64_t lda, int64_t m, int64_t d, int64_t col, int64_t w,
                    double* d_tau, QrRefl& Rf, cudaStream_t st) {
  CKR(qr_refl_alloc(Rf, m - d, (int)w));
  const int64_t smax = (int64_t)std::min<size_t>(c.smem_optin, 227 * 1024) - 1024;
  const int gcap = std::min(c.sms, QR_MAXG);
  for (int64_t p0 = 0; p0 < w; p0 += QR_LW) {
    const int lw = (int)std::min<int64_t>(QR_LW, w - p0);
    const int64_t r0 = d + p0, mp = m - r0;
    int R = (int)std::max<int64_t>(g_qr_rows > 0 ? g_qr_rows : 512, (mp + gcap - 1) / gcap);
    int G = (int)((mp + R - 1) / R);
    R = (int)((mp + G - 1) / G);
    // one thread-block cluster when the leaf fits 16 CTAs' shared memory
    const int64_t clx = (int64_t)(2 * QR_CL_MAX * QR_LW + 2 * QR_LW) * 8;
    bool cl = false;
    if (g_qr_cluster) {
      int Rc = (int)std::max<int64_t>(g_qr_rows > 0 ? g_qr_rows : 512, (mp + QR_CL_MAX - 1) / QR_CL_MAX);
      const int Gc = (int)((mp + Rc - 1) / Rc);
      Rc = (int)((mp + Gc - 1) / Gc);
      if (Gc <= QR_CL_MAX && (int64_t)std::max(Rc, 2 * QR_LW) * QR_LDT * 8 + clx <= smax) {
        cl = true;
        R = Rc;
        G = Gc;
      }
    }
    if ((int64_t)R * QR_LDT * 8 > smax) return set_err(PFLU_ERR_UNSUPPORTED, "QR panel of %lld rows too tall", (long long)mp);
    if (G > QR_MAXG || G > c.sms) return set_err(PFLU_ERR_UNSUPPORTED, "QR panel grid %d too large", G);
    QrLeafArgs la;
    la.a = a; la.lda = lda; la.r0 = r0; la.m = m; la.c0 = col + p0; la.w = lw;
    la.G = G; la.R = R;
    la.tau = d_tau + p0;
    la.dots = q.leafx;
    la.drow = q.leafx + 2 * QR_MAXG * QR_LW;
    la.gram = q.leafx + 2 * QR_MAXG * QR_LW + 64;
    la.bar = q.bar;
    la.vd = Rf.vd.p; la.ldv = Rf.ldv;
    la.vt = Rf.vt.p; la.ldvt = Rf.ldvt;
    la.tt = Rf.tt.p; la.ldt = Rf.ldt;
    la.p0 = (int)p0;
    void* args[] = {&la};
    if (cl) {
      const size_t smem = (size_t)std::max(R, 2 * QR_LW) * QR_LDT * 8 + (size_t)clx;
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(QR_THREADS);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CK(cudaLaunchKernelExC(&cfg, (const void*)qr_leaf_kernel<true>, args));
    } else {
      CK(cudaMemsetAsync(q.bar, 0, sizeof(unsigned), st));
      const size_t smem = (size_t)std::max(R, 2 * QR_LW) * QR_LDT * 8;
      CK(cudaLaunchCooperativeKernel((void*)qr_leaf_kernel<false>, dim3(G), dim3(QR_THREADS), args, smem, st));
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const int64_t rest = w - p0 - lw;
    if (rest > 0) {
      const QrView v = {Rf.vd.p + p0 * Rf.ldv + p0, Rf.ldv, Rf.vt.p + p0 * Rf.ldvt + p0, Rf.ldvt,
                        Rf.tt.p + p0 * Rf.ldt + p0, Rf.ldt, mp, lw};
      CKR(qr_apply(c, q.ws[0], v, a + r0 * lda + col + p0 + lw, lda, rest, st));
    }
  }
  return PFLU_OK;
}

// Blocked QR, depth 0 (dmf_mtb order) or 1 (dmf_la: TU_L(k) + PF(k+1) on the panel stream while
// TU_R(k) runs on the trailing stream), asynchronous; the caller's stream `st` is joined at the end.
using RowSinkM = std::function<int(int64_t r0, int64_t r1, const std::vector<cudaEvent_t>& after)>;
static int geqrf_host_chunked(DevCtx& c, double* a, int64_t m, int64_t n, int64_t lda, int64_t b, double* d_tau,
                              cudaStream_t st, const double* ha, int64_t hlda, int chunks, const RowSinkM& sinkm);
static int g_qr_chunks = []() { const char* e = getenv("PFLU_QR_CHUNKS"); return e ? atoi(e) : 6; }();

// `sink` (optional, host-buffer calls): row block k is final once step k's updates (TU_R(k) and
// TU_L(k)) are done -- later steps only touch rows >= (k+1) b -- and is handed to the sink then.
static int geqrf_async(DevCtx& c, double* a, int64_t m, int64_t n, int64_t lda, int64_t b, int lookahead,
                       double* d_tau, cudaStream_t st, const RowSink* sink = nullptr, Tracer* trp = nullptr) {
  Tracer tr_off;
  Tracer& tr = trp ? *trp : tr_off;
  QrCtx* qp = nullptr;
  CKR(qr_ctx(c, &qp));
  QrCtx& q = *qp;
  const int64_t steps = (n + b - 1) / b;
  {  // every workspace at its maximum size before the first launch (see QrBuf::need)
    const int64_t bb = std::min(b, n);
    for (QrRefl* R : {&q.refl[0], &q.refl[1]}) {
      CKR(R->vd.need((size_t)(m * qr_even(bb))));
      CKR(R->vt.need((size_t)(bb * qr_even(m))));
      CKR(R->tt.need((size_t)(bb * qr_even(bb))));
    }
    for (auto& w : q.ws) {
      CKR(w.w.need((size_t)(bb * qr_even(n))));
      CKR(w.z.need((size_t)(bb * qr_even(n))));
      CKR(w.g.need((size_t)(bb * qr_even(bb))));
      CKR(w.part.need((size_t)4 * c.sms * 128 * 65));  // split-K slices: S * M * ldp <= 4 sms * 128 * 65
    }
  }
  cudaStream_t sP = c.sP, sU = c.sU;
  CKR(ctx_events(c, 5));
  cudaEvent_t e_in = c.ev[0], e_pf = c.ev[1], e_tu = c.ev[2], e_out = c.ev[3], e_tl = c.ev[4];
  CK(cudaEventRecord(e_in, st));
  CK(cudaStreamWaitEvent(sP, e_in, 0));
  CK(cudaStreamWaitEvent(sU, e_in, 0));
  CKR(tr.start(sP));
  auto bw_of = [&](int64_t k) { return std::min(b, n - k * b); };
  // PF(k) on the panel stream: leaves + in-panel block reflectors (+ T when a trailing update follows)
  auto pf = [&](int64_t k, bool with_t) -> int {
    const int64_t col0 = k * b, bw = bw_of(k);
    QrRefl& R = q.refl[k & 1];
    int t_pf = -1;
    CKR(tr.begin(PFLU_TRACE_PF, (int)k, sP, &t_pf));
    CKR(qr_panel(c, q, a, lda, m, col0, col0, bw, d_tau + col0, R, sP));
    if (with_t) CKR(qr_finish_t(c, q.ws[0], R, d_tau + col0, sP));
    return tr.end(t_pf, sP);
  };
  if (lookahead == 0) {
    for (int64_t k = 0; k < steps; ++k) {
      const int64_t col0 = k * b, bw = bw_of(k), lo = col0 + bw;
      QrRefl& R = q.refl[k & 1];
      CKR(pf(k, lo < n));
      if (lo < n) {
        int t_tu = -1;
        CKR(tr.begin(PFLU_TRACE_TU, (int)k, sP, &t_tu));
        CKR(qr_apply(c, q.ws[0], qr_view(R), a + col0 * lda + lo, lda, n - lo, sP));
        CKR(tr.end(t_tu, sP));
      }
      if (sink) CKR((*sink)(col0, col0 + bw, sP));
    }
    CK(cudaEventRecord(e_out, sP));
    CK(cudaStreamWaitEvent(st, e_out, 0));
    return PFLU_OK;
  }
  // look-ahead 1 (device buffers): the column-chunk schedule of geqrf_host_chunked without the H2D
  if (g_qr_chunks > 1 && !sink && !tr.on && b < n)
    return geqrf_host_chunked(c, a, m, n, lda, b, d_tau, st, nullptr, 0, g_qr_chunks, RowSinkM());
  CKR(pf(0, bw_of(0) < n));
  for (int64_t k = 0; k < steps; ++k) {
    const int64_t col0 = k * b, bw = bw_of(k), lo = col0 + bw;
    if (lo >= n) break;
    QrRefl& R = q.refl[k & 1];
    CK(cudaEventRecord(e_pf, sP));
    // TU_R(k): columns beyond block k+1, on the trailing stream
    const int64_t lo2 = lo + bw_of(k + 1);
    if (lo2 < n) {
      CK(cudaStreamWaitEvent(sU, e_pf, 0));
      int t_r = -1;
      CKR(tr.begin(PFLU_TRACE_TU_R, (int)k, sU, &t_r));
      CKR(qr_apply(c, q.ws[1], qr_view(R), a + col0 * lda + lo2, lda, n - lo2, sU));
      CKR(tr.end(t_r, sU));
    }
    // TU_L(k) + PF(k+1) on the panel stream; TU_R(k-1) (recorded before e_tu is re-recorded
    // below) finished updating block k+1
    int t_l = -1;
    CKR(tr.begin(PFLU_TRACE_TU_L, (int)k, sP, &t_l));
    CKR(qr_apply(c, q.ws[0], qr_view(R), a + col0 * lda + lo, lda, bw_of(k + 1), sP));
    CKR(tr.end(t_l, sP));
    if (sink) {  // row block k: final after TU_L(k) (panel stream) and TU_R(k) (trailing stream)
      CK(cudaEventRecord(e_tl, sP));
      CK(cudaStreamWaitEvent(sU, e_tl, 0));
      CKR((*sink)(col0, col0 + bw, sU));
    }
    CKR(pf(k + 1, lo + bw_of(k + 1) < n));
    // the next TU_L / build (which rewrites refl[(k+1)&1] ... refl[k&1] at step k+2) must follow TU_R(k)
    if (lo2 < n) {
      CK(cudaEventRecord(e_tu, sU));
      CK(cudaStreamWaitEvent(sP, e_tu, 0));
    }
  }
  CK(cudaEventRecord(e_out, sU));
  CK(cudaStreamWaitEvent(st, e_out, 0));
  CK(cudaEventRecord(e_out, sP));
  CK(cudaStreamWaitEvent(st, e_out, 0));
  return PFLU_OK;
}

// pflu_geqrf, look-ahead 1, host source: the H2D is issued per column chunk (the first two block
// columns first) and the trailing update of every step runs per chunk on that chunk's stream, waiting
// only for its own columns, so later columns are still in flight while the first steps run.  A chunk
// that arrives late catches up on every earlier step, so the reflectors of the last RING steps are
// kept (the panel stream waits before reusing a ring slot).  Row block k is handed to `sinkm` once
// TU_L(k) and every chunk's TU_R(k) are done.
static int geqrf_host_chunked(DevCtx& c, double* a, int64_t m, int64_t n, int64_t lda, int64_t b, double* d_tau,
                              cudaStream_t st, const double* ha, int64_t hlda, int chunks, const RowSinkM& sinkm) {
  QrCtx* qp = nullptr;
  CKR(qr_ctx(c, &qp));
  QrCtx& q = *qp;
  constexpr int NR = QrCtx::RING;
  const int64_t steps = (n + b - 1) / b;
  auto bw_of = [&](int64_t k) { return std::min(b, n - k * b); };
  // chunks in block units: chunk 0 = blocks [0, 2), the rest split evenly
  std::vector<int64_t> blo, bhi;
  blo.push_back(0);
  bhi.push_back(std::min<int64_t>(2, steps));
  const int rest_ch = std::max(0, std::min<int>(chunks - 1, (int)(steps - bhi[0])));
  for (int i = 0; i < rest_ch; ++i) {
    const int64_t rb = steps - bhi[0];
    blo.push_back(bhi[0] + rb * i / rest_ch);
    bhi.push_back(bhi[0] + rb * (i + 1) / rest_ch);
  }
  const int nch = (int)blo.size();
  auto chunk_of = [&](int64_t blk) { int ci = 0; while (ci + 1 < nch && blk >= bhi[ci]) ++ci; return ci; };
  {  // every buffer at its maximum before the first launch (see QrBuf::need)
    for (auto& R : q.ring) {
      CKR(R.vd.need((size_t)(m * qr_even(b))));
      CKR(R.vt.need((size_t)(b * qr_even(m))));
      CKR(R.tt.need((size_t)(b * qr_even(b))));
    }
    for (QrScratch* w : {&q.ws[0], &q.wsc[0], &q.wsc[1], &q.wsc[2], &q.wsc[3], &q.wsc[4], &q.wsc[5], &q.wsc[6],
                         &q.wsc[7]}) {
      CKR(w->w.need((size_t)(b * qr_even(n))));
      CKR(w->z.need((size_t)(b * qr_even(n))));
      CKR(w->g.need((size_t)(b * qr_even(b))));
      CKR(w->part.need((size_t)4 * c.sms * 128 * 65));
    }
  }
  // events: [0] start, [1 + ci] H2D of chunk ci, then per step: e_pf, e_tl, nch chunk events
  const size_t ne = 2 + (size_t)nch;
  CKR(ctx_events(c, 1 + nch + (size_t)steps * ne + 1));
  cudaEvent_t e_in = c.ev[0];
  auto evH = [&](int ci) { return c.ev[1 + ci]; };
  auto evPF = [&](int64_t k) { return c.ev[1 + nch + (size_t)k * ne]; };
  auto evTL = [&](int64_t k) { return c.ev[1 + nch + (size_t)k * ne + 1]; };
  auto evC = [&](int64_t k, int ci) { return c.ev[1 + nch + (size_t)k * ne + 2 + ci]; };
  cudaEvent_t e_end = c.ev[1 + nch + (size_t)steps * ne];
  cudaStream_t sP = c.sP;
  CK(cudaEventRecord(e_in, st));
  CK(cudaStreamWaitEvent(sP, e_in, 0));
  for (int ci = 0; ci < nch; ++ci) {
    const int64_t c0 = blo[ci] * b, c1 = std::min(n, bhi[ci] * b);
    if (ha)
      CK(cudaMemcpy2DAsync(a + c0, lda * 8, ha + c0, hlda * 8, (c1 - c0) * 8, m, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(evH(ci), st));
    CK(cudaStreamWaitEvent(c.sC[ci], e_in, 0));
  }
  auto pf = [&](int64_t k) -> int {
    const int64_t col0 = k * b, bw = bw_of(k);
    QrRefl& R = q.ring[k % NR];
    CKR(qr_panel(c, q, a, lda, m, col0, col0, bw, d_tau + col0, R, sP));
    if (col0 + bw < n) CKR(qr_finish_t(c, q.ws[0], R, d_tau + col0, sP));
    return PFLU_OK;
  };
  CK(cudaStreamWaitEvent(sP, evH(0), 0));
  CKR(pf(0));
  for (int64_t k = 0; k < steps; ++k) {
    const int64_t col0 = k * b, bw = bw_of(k), lo = col0 + bw;
    if (lo >= n) break;
    QrRefl& R = q.ring[k % NR];
    CK(cudaEventRecord(evPF(k), sP));
    const int64_t lo2 = lo + bw_of(k + 1);
    for (int ci = 0; ci < nch; ++ci) {  // TU_R(k), chunk by chunk
      cudaStream_t sc = c.sC[ci];
      const int64_t c0 = std::max(lo2, blo[ci] * b), c1 = std::min(n, bhi[ci] * b);
      if (c1 > c0) {
        CK(cudaStreamWaitEvent(sc, evH(ci), 0));
        CK(cudaStreamWaitEvent(sc, evPF(k), 0));
        CKR(qr_apply(c, q.wsc[ci], qr_view(R), a + col0 * lda + c0, lda, c1 - c0, sc));
      }
      CK(cudaEventRecord(evC(k, ci), sc));
    }
    // TU_L(k): block k+1 was last updated by TU_R(k-1) on its chunk
    const int cb = chunk_of(k + 1);
    CK(cudaStreamWaitEvent(sP, k >= 1 ? evC(k - 1, cb) : evH(cb), 0));
    CKR(qr_apply(c, q.ws[0], qr_view(R), a + col0 * lda + lo, lda, bw_of(k + 1), sP));
    CK(cudaEventRecord(evTL(k), sP));
    // PF(k+1) reuses ring slot (k+1) % NR: every chunk must be done with step k+1-NR
    if (k + 1 - NR >= 0)
      for (int ci = 0; ci < nch; ++ci) CK(cudaStreamWaitEvent(sP, evC(k + 1 - NR, ci), 0));
    CKR(pf(k + 1));
    std::vector<cudaEvent_t> fin{evTL(k)};
    for (int ci = 0; ci < nch; ++ci) fin.push_back(evC(k, ci));
    if (sinkm) CKR(sinkm(col0, col0 + bw, fin));
  }
  for (int ci = 0; ci < nch; ++ci) {
    CK(cudaEventRecord(e_end, c.sC[ci]));
    CK(cudaStreamWaitEvent(st, e_end, 0));
  }
  CK(cudaEventRecord(e_end, sP));
  CK(cudaStreamWaitEvent(st, e_end, 0));
  return PFLU_OK;
}

}  // namespace pflu
