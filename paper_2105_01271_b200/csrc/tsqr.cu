// K4: Householder TSQR for tall-skinny matrices (<= 32 columns per panel).
//
// Replaces thin_qr / np.linalg.qr (src/kernels.py:74-84) on the path.  The
// sketch bases on this path are numerically rank deficient (SURVEY.md 7 "Hard
// parts"): CholeskyQR breaks down, so orthogonalisation is Householder
// based, which keeps the span of every direction to eps * ||X|| regardless of
// conditioning.
//
// Factor (tsqr_leaf_kernel): a CTA factors a 256 x cols chunk with
// LANE = COLUMN: warp w holds rows g = 8 i + w (register slot i) and lane c
// holds those 32 entries of column c.  Householder step j needs ONE block
// reduction: lane j's column reaches the other lanes of its warp by shuffles,
// and the vector of dot products <x_j(below j), x_c> -- whose j-th entry is
// the norm^2 below the diagonal -- is reduced across the 8 warps together
// with row j (double-buffered, one __syncthreads per step).  The same dot
// products give v_c^T v_j for c < j, from which the compact-WY factor T
// (H_0 ... H_{n-1} = I - V T V^T) is formed in the CTA at the end.
// The chunks' R factors (cols x cols) are stacked and factored again until a
// single chunk remains; its R, sign-normalised to diag(R) >= 0, is the result.
//
// Q (tsqr_apply_kernel, top-down): each chunk's block of the parent Q is
// Q_h [B_h; 0] = [B_h; 0] - V_h (T_h (V_top,h^T B_h)), a parallel 64-row-tile
// product (no per-reflector synchronisation); the root starts from
// B = diag(sign(R_jj)).  Fixed reduction orders throughout: bitwise
// reproducible.
#include "async.cuh"
#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

#include <cooperative_groups.h>
#include <vector>

namespace cg = cooperative_groups;

namespace spb {

int gemm(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
         cudaStream_t s);

constexpr int kQB = 32;                 // panel width (register columns)
constexpr int kQWarps = 8;
constexpr int kQThreads = kQWarps * 32;
constexpr int kQCH = kQWarps * 32;      // rows per CTA
constexpr int kQMaxCluster = 16;        // CTAs per chunk (non-portable cluster size)
constexpr int kQSlotsTall = 40;         // register slots per lane of the 320-row leaf variant

// Row mapping: local row g = 8*i + w lives in warp w, register slot i, so
// the 32 diagonal rows are spread 4 per warp (slots 0..3): only those slots
// need j-dependent masks, every other slot is strictly below every diagonal.
__device__ __forceinline__ int qrow(int i, int w) { return i * kQWarps + w; }
constexpr int kQDiagSlots = kQB / kQWarps;  // 4

// Factor chunk h of X (rows x cols).  A chunk is one thread-block CLUSTER of
// `cl` CTAs (cl * 256 rows): every CTA reduces its 8 warps' partial dot
// products, pushes the 32-vector to every CTA of the cluster through
// distributed shared memory, and after one cluster barrier all CTAs sum the
// cl partials in rank order -- identical scalars everywhere, one cluster
// barrier per Householder step, and one level of the tree for up to 4096
// rows.  Writes the reflectors (strictly below the chunk diagonal, unit
// diagonal implicit) to V (rows x 32), the chunk's 32 x 32 compact-WY factor
// to Tg, and its cols x cols upper-triangular R to Rs[h * cols ..) (ld 32).
// When Rfinal != nullptr (single chunk = root) R is also written there with
// diag(R) >= 0 and the row signs to sgn.
template <int NS>  // register slots per lane: a CTA holds 8 NS rows (NS = 32: 256, NS = 40: 320)
__global__ void __launch_bounds__(kQThreads)
tsqr_leaf_kernel(const double* __restrict__ X, int64_t rows, int cols, int64_t ldx, double* __restrict__ V,
                 double* __restrict__ Tg, double* __restrict__ Rs, double* __restrict__ Rfinal, int64_t ldr,
                 double* __restrict__ sgn, double* __restrict__ Mg) {
  SPB_PDL_ENTRY();
  __shared__ double red[2][kQWarps][kQB];
  __shared__ double rowj[2][kQB];
  __shared__ double cbuf[2][kQMaxCluster][kQB];  // cluster partials (pushed by peers)
  __shared__ double crow[2][kQB];                // row j (pushed by rank 0)
  __shared__ __align__(8) uint64_t cbar[2];      // tx-counted arrival of a step's pushes
  __shared__ double zs[kQB][kQB + 1];  // zs[c][j] = v_c^T v_j (c < j)
  __shared__ double ts[kQB][kQB + 1];  // T (upper triangular)
  __shared__ double tau_s[kQB], inv_s[kQB], beta_s[kQB];
  __shared__ __align__(16) double colb[kQWarps][NS];
  constexpr int CH = NS * kQWarps;  // rows per CTA
  cg::cluster_group cluster = cg::this_cluster();
  const int cl = (int)cluster.num_blocks();
  const int cr = (int)cluster.block_rank();
  const int w = threadIdx.x >> 5, c = threadIdx.x & 31;
  const int64_t h = blockIdx.x / cl;
  const int64_t chunk0 = h * (int64_t)cl * CH;
  const int64_t c0 = chunk0 + (int64_t)cr * CH;  // my first row
  const int nrow = (int)std::max<int64_t>(0, imin64(CH, rows - c0));
  const int chunk_rows = (int)imin64((int64_t)cl * CH, rows - chunk0);
  const bool top = cr == 0;  // rows 0..31 of the chunk live in rank 0
  double x[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    const int g = qrow(i, w);
    x[i] = (g < nrow && c < cols) ? X[(c0 + g) * ldx + c] : 0.0;
  }
  const int nref = chunk_rows < cols ? chunk_rows : cols;
  for (int e = threadIdx.x; e < kQB * (kQB + 1); e += kQThreads) (&zs[0][0])[e] = 0.0;
  // per step every CTA receives cl partial vectors and row j: (cl + 1) * 256 bytes
  const uint32_t step_bytes = (uint32_t)(cl + 1) * kQB * sizeof(double);
  if (cl > 1) {
    if (threadIdx.x == 0) {
      mbar_init(&cbar[0], 1);
      mbar_init(&cbar[1], 1);
      mbar_fence_init();
      mbar_arrive_expect_tx(&cbar[0], step_bytes);
      mbar_arrive_expect_tx(&cbar[1], step_bytes);
    }
    cluster.sync();  // barriers initialised before any peer pushes
  }
  // Column j is left untouched by its own step (it keeps alpha_j on the
  // diagonal and (alpha_j - beta_j) v_j below it); the scaled reflector and
  // beta_j are substituted when the chunk is written out.  Steps therefore
  // update columns c > j only, uniformly across the warp:
  //   x_c -= x_j * (inv_j * w_c),  w_c = tau_j v_j^T x_c.
  int buf = 0;
#ifdef SPB_TSQR_TRACE
  long long tr_a = 0, tr_b = 0, tr_c = 0, tr_beg = clock64(), tr_s0, tr_s1, tr_s2;
#endif
  for (int j = 0; j < nref; ++j) {
#ifdef SPB_TSQR_TRACE
    tr_s0 = clock64();
#endif
    // (1) lane j publishes its column (my warp's rows) through shared memory;
    // partial <x_j, x_c> over my rows
    if (c == j) {
#pragma unroll
      for (int i = 0; i < NS; i += 2) *reinterpret_cast<double2*>(&colb[w][i]) = make_double2(x[i], x[i + 1]);
    }
    __syncwarp();
    double xj[NS];
#pragma unroll
    for (int i = 0; i < NS; i += 2) {
      const double2 t = *reinterpret_cast<const double2*>(&colb[w][i]);
      xj[i] = t.x;
      xj[i + 1] = t.y;
    }
    if (top) {
#pragma unroll
      for (int i = 0; i < kQDiagSlots; ++i)
        if (qrow(i, w) <= j) xj[i] = 0.0;
    }
    double pa[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) pa[u] = xj[u] * x[u];
#pragma unroll
    for (int i = 8; i < NS; i += 8)
#pragma unroll
      for (int u = 0; u < 8; ++u) pa[u] = fma(xj[i + u], x[i + u], pa[u]);
    red[buf][w][c] = ((pa[0] + pa[1]) + (pa[2] + pa[3])) + ((pa[4] + pa[5]) + (pa[6] + pa[7]));
    const int jw = j & (kQWarps - 1), js = j >> 3;  // owner warp / slot of row j (rank 0)
    if (top && w == jw) {
      double rj = x[0];
#pragma unroll
      for (int i = 1; i < kQDiagSlots; ++i)
        if (i == js) rj = x[i];
      rowj[buf][c] = rj;
    }
    __syncthreads();
#ifdef SPB_TSQR_TRACE
    tr_s1 = clock64();
    tr_a += tr_s1 - tr_s0;
#endif
    // (2) reflector scalars (every thread of the cluster, same order: identical values)
    double dc, sigma2, alpha, ac;
    {
      double rc[kQWarps], rq[kQWarps];
#pragma unroll
      for (int q = 0; q < kQWarps; ++q) {
        rc[q] = red[buf][q][c];
        rq[q] = red[buf][q][j];
      }
      dc = ((rc[0] + rc[1]) + (rc[2] + rc[3])) + ((rc[4] + rc[5]) + (rc[6] + rc[7]));
      sigma2 = ((rq[0] + rq[1]) + (rq[2] + rq[3])) + ((rq[4] + rq[5]) + (rq[6] + rq[7]));
    }
    if (cl > 1) {
      {
        // the pushes are spread over the warps (warp w serves ranks w, w + 8):
        // one or two remote stores per lane instead of cl from warp 0 alone
        const double rv = top ? rowj[buf][c] : 0.0;
        for (int d = w; d < cl; d += kQWarps) {
          const uint32_t bar = cluster_addr(&cbar[buf], d);
          st_async_f64(cluster_addr(&cbuf[buf][cr][c], d), dc, bar);
          if (top) st_async_f64(cluster_addr(&crow[buf][c], d), rv, bar);
        }
      }
      mbar_wait_cluster(&cbar[buf], (uint32_t)(j >> 1) & 1u);
      // re-arm this buffer for step j + 2 (every thread has passed the wait
      // of step j - 1 on the other buffer, and reads of step j happen before
      // the __syncthreads of step j + 1, which precedes any push of step j + 2
      // by this CTA's peers)
      // rank order in 4 interleaved sums (same in every CTA); cl is a power of 2
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
      int d = 0;
      for (; d + 3 < cl; d += 4) {
        a0 += cbuf[buf][d][c];
        a1 += cbuf[buf][d + 1][c];
        a2 += cbuf[buf][d + 2][c];
        a3 += cbuf[buf][d + 3][c];
        g0 += cbuf[buf][d][j];
        g1 += cbuf[buf][d + 1][j];
        g2 += cbuf[buf][d + 2][j];
        g3 += cbuf[buf][d + 3][j];
      }
      for (; d < cl; ++d) {
        a0 += cbuf[buf][d][c];
        g0 += cbuf[buf][d][j];
      }
      dc = (a0 + a1) + (a2 + a3);
      sigma2 = (g0 + g1) + (g2 + g3);
      alpha = crow[buf][j];
      ac = crow[buf][c];
      if (threadIdx.x == 0) mbar_arrive_expect_tx(&cbar[buf], step_bytes);
    } else {
      alpha = rowj[buf][j];
      ac = rowj[buf][c];
    }
#ifdef SPB_TSQR_TRACE
    tr_s2 = clock64();
    tr_b += tr_s2 - tr_s1;
#endif
    double beta = alpha, tj = 0.0, inv = 0.0;
    if (sigma2 > 0.0) {
      // one rsqrt and one division: nrm = s2 / sqrt(s2), tau = -(alpha - beta) / beta
      const double s2 = fma(alpha, alpha, sigma2);
      const bool fr = fast_range(s2);
      const double rs = fr ? fast_rsqrt(s2) : rsqrt(s2);
      const double sg = alpha >= 0.0 ? 1.0 : -1.0;
      beta = -sg * (s2 * rs);
      const double dd = alpha - beta;  // |dd| >= ||x_j(j:)|| > 0
      inv = fr ? fast_rcp(dd) : 1.0 / dd;
      tj = sg * dd * rs;
    }
    const double vv = fma(inv, dc, ac);  // v_j^T x_c (c > j);  (alpha_c - beta_c) v_c^T v_j (c < j)
    // (3) apply H_j to the trailing columns
    const double wc = c > j ? tj * vv : 0.0;
    const double sc = inv * wc;
#pragma unroll
    for (int i = 0; i < NS; ++i) x[i] = fma(-xj[i], sc, x[i]);
    if (top && w == jw) {
#pragma unroll
      for (int i = 0; i < kQDiagSlots; ++i)
        if (i == js) x[i] -= wc;
    }
    if (c < j && w == 0) zs[c][j] = inv_s[c] * vv;
    if (threadIdx.x == 0) {
      tau_s[j] = tj;
      inv_s[j] = inv;
      beta_s[j] = beta;
    }
    buf ^= 1;
#ifdef SPB_TSQR_TRACE
    tr_c += clock64() - tr_s2;
#endif
  }
#ifdef SPB_TSQR_TRACE
  if (threadIdx.x == 0 && blockIdx.x < cl)
    printf("tsqr_leaf rows=%lld cl=%d rank=%d steps=%d: loop %lld cyc; per step dots+sync %lld, exchange %lld, scalars+update %lld\n",
           (long long)rows, cl, cr, nref, clock64() - tr_beg, tr_a / nref, tr_b / nref, tr_c / nref);
#endif
  if (cl > 1) cluster.sync();  // no CTA leaves while peers' pushes are in flight
  __syncthreads();
  // reflectors (coalesced rows)
  const double inv_c = c < nref ? inv_s[c] : 0.0;
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    const int g = qrow(i, w);
    const int gc = cr * CH + g;  // chunk-local row
    if (g < nrow) V[(c0 + g) * kQB + c] = (gc > c && c < nref) ? x[i] * inv_c : 0.0;
  }
  if (!top) return;
  // root with Mg: keep V_top (reflector rows 0..31, unit diagonal) for M below
  __shared__ double vtop_s[kQB][kQB + 1];
  __shared__ double sg_s[kQB];
  if (Mg != nullptr) {
#pragma unroll
    for (int i = 0; i < kQDiagSlots; ++i) {
      const int g = qrow(i, w);
      vtop_s[g][c] = c < nref ? (g > c ? x[i] * inv_c : (g == c ? 1.0 : 0.0)) : 0.0;
    }
  }
  // compact-WY T by recursive doubling: for adjacent blocks [V1 V2] of width
  // b, T12 = -T11 (V1^T V2) T22 (exact for tau = 0 too); 5 levels of two
  // parallel small products instead of a 32-step serial recurrence.
  for (int e = threadIdx.x; e < kQB * kQB; e += kQThreads) {
    const int r = e / kQB, q = e % kQB;
    ts[r][q] = (r == q && q < nref) ? tau_s[q] : 0.0;
  }
  __syncthreads();
  double* wsm = &red[0][0][0];  // 16 b <= 256 products per level
  for (int b = 1; b < kQB; b <<= 1) {
    const int nout = (kQB / 2) * b;
    if (threadIdx.x < nout) {
      const int e = threadIdx.x, p = e / (b * b), rq = e % (b * b), r = rq / b, q = rq % b;
      const int o1 = p * 2 * b, o2 = o1 + b;
      double a = 0.0;
      for (int l = 0; l <= q; ++l) a = fma(zs[o1 + r][o2 + l], ts[o2 + l][o2 + q], a);
      wsm[e] = a;
    }
    __syncthreads();
    if (threadIdx.x < nout) {
      const int e = threadIdx.x, p = e / (b * b), rq = e % (b * b), r = rq / b, q = rq % b;
      const int o1 = p * 2 * b, o2 = o1 + b;
      double a = 0.0;
      for (int l = r; l < b; ++l) a = fma(ts[o1 + r][o1 + l], wsm[p * b * b + l * b + q], a);
      ts[o1 + r][o2 + q] = -a;
    }
    __syncthreads();
  }
  // R rows (rank 0 holds chunk rows 0..31), T
#pragma unroll
  for (int i = 0; i < kQDiagSlots; ++i) {
    const int g = qrow(i, w);  // g < 32
    if (g < cols) {
      double rv = (g < nrow && c >= g && c < cols) ? x[i] : 0.0;
      if (c == g && g < nref) rv = beta_s[g];
      x[i] = rv;
      Rs[(h * cols + g) * kQB + c] = rv;
    }
  }
  for (int e = threadIdx.x; e < kQB * kQB; e += kQThreads) Tg[h * kQB * kQB + e] = ts[e / kQB][e % kQB];
  if (Rfinal != nullptr) {
    // root: rows of R with diag(R) >= 0 (the diagonal sits in warp g & 7, slot g >> 3)
#pragma unroll
    for (int i = 0; i < kQDiagSlots; ++i) {
      const int g = qrow(i, w);
      if (g < cols) {
        const double d = __shfl_sync(0xffffffffu, x[i], g);
        const double sg = d < 0.0 ? -1.0 : 1.0;
        if (c < cols) Rfinal[(int64_t)g * ldr + c] = (c >= g) ? sg * x[i] : 0.0;
        if (c == 0) {
          sgn[g] = sg;
          sg_s[g] = sg;
        }
      }
    }
    if (Mg != nullptr) {
      // M = T V_top^T diag(sgn) (the root's Q = [diag(sgn); 0] - V M), so the
      // Q pass (tsqr_q_kernel) is one small product per row
      __syncthreads();
      for (int e = threadIdx.x; e < kQB * kQB; e += kQThreads) {
        const int k = e / kQB, cc = e % kQB;
        double a = 0.0;
        if (cc < cols) {
          for (int l = k; l < kQB; ++l) a = fma(ts[k][l], vtop_s[cc][l], a);
          a *= sg_s[cc];
        }
        Mg[e] = a;
      }
    }
  }
}

// Q of a single-chunk TSQR: rows [0, rows) of Q = [diag(sgn); 0] - V M, M from
// the root leaf (32 x 32).  CTA = 64 rows; thread (row, 8-column group).
__global__ void __launch_bounds__(kQThreads)
tsqr_q_kernel(const double* __restrict__ V, const double* __restrict__ Mg, const double* __restrict__ sgn,
              int64_t rows, int cols, double* __restrict__ Q, int64_t ldq) {
  SPB_PDL_ENTRY();
  constexpr int P = kQB + 1;
  __shared__ double ms[kQB * P];
  __shared__ double vs[64 * P];
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * 64;
  const int nr = (int)imin64(64, rows - r0);
  for (int e = t; e < kQB * kQB; e += kQThreads) cp_async_f64(&ms[(e / kQB) * P + (e % kQB)], Mg + e, true);
  for (int e = t; e < 64 * kQB; e += kQThreads) {
    const int g = e / kQB, k = e % kQB;
    cp_async_f64(&vs[g * P + k], V + (r0 + (g < nr ? g : 0)) * kQB + k, g < nr);
  }
  cp_async_wait_all();
  __syncthreads();
  if (r0 < kQB && t < nr && r0 + t < kQB) vs[t * P + r0 + t] = 1.0;  // implicit unit diagonal
  __syncthreads();
  const int g = t >> 2, c0 = (t & 3) * 8;
  if (g >= nr) return;
  double acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = 0.0;
#pragma unroll 8
  for (int k = 0; k < kQB; ++k) {
    const double v = vs[g * P + k];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = fma(v, ms[k * P + c0 + u], acc[u]);
  }
  const int64_t gr = r0 + g;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int cc = c0 + u;
    if (cc < cols) Q[gr * ldq + cc] = (gr == cc ? sgn[cc] : 0.0) - acc[u];
  }
}

// Top-down Q formation for chunk h = blockIdx.x / tiles (chunk_rows rows),
// rows tile (blockIdx.x % tiles) * 64 of it:  Out = [B_h; 0] - V_h M_h,
// M_h = T_h (V_top^T B_h), B_h = Bin[h * cols ..) (cols x cols, ld 32) or
// diag(sgn) at the root.  Out has cols columns.
constexpr int kApRows = 64;

__global__ void __launch_bounds__(kQThreads)
tsqr_apply_kernel(const double* __restrict__ V, const double* __restrict__ Tg, int64_t rows, int cols,
                  int chunk_rows, const double* __restrict__ Bin, const double* __restrict__ sgn,
                  double* __restrict__ Out, int64_t ldo) {
  SPB_PDL_ENTRY();
  constexpr int P = kQB + 1;
  __shared__ double ub[kApRows * P];  // V_top | B_h, later the V rows of the tile
  __shared__ double tsm[kQB * P];     // T_h
  __shared__ double ws[kQB * P];      // V_top^T B, then M
  double* vt = ub;
  double* bs = ub + kQB * P;
  double* vr = ub;
  const int tiles = chunk_rows / kApRows;
  const int h = blockIdx.x / tiles, tile = blockIdx.x % tiles;
  const int64_t c0 = (int64_t)h * chunk_rows;
  const int nrow = (int)imin64(chunk_rows, rows - c0);
  const int r0 = tile * kApRows;
  if (r0 >= nrow) return;  // uniform per CTA
  const int nr = nrow - r0 < kApRows ? nrow - r0 : kApRows;
  const int tid = threadIdx.x;
  auto b_at = [&](int g, int k) -> double {
    if (g >= cols || k >= cols) return 0.0;
    return Bin ? Bin[((int64_t)h * cols + g) * kQB + k] : (g == k ? sgn[g] : 0.0);
  };
  // reflectors carry an implicit unit diagonal (stored zeros on/above it)
  for (int e = tid; e < kQB * kQB; e += kQThreads) {
    const int g = e / kQB, k = e % kQB;
    cp_async_f64(&vt[g * P + k], V + (c0 + (g < nrow ? g : 0)) * kQB + k, g < nrow);
    cp_async_f64(&tsm[g * P + k], Tg + (int64_t)h * kQB * kQB + e, true);
    if (Bin) {
      const bool ok = g < cols && k < cols;
      cp_async_f64(&bs[g * P + k], ok ? Bin + ((int64_t)h * cols + g) * kQB + k : Bin, ok);
    } else {
      bs[g * P + k] = b_at(g, k);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  if (tid < kQB && tid < nrow) vt[tid * P + tid] = 1.0;
  __syncthreads();
  // W = V_top^T B  (only the top cols rows of [B; 0] are nonzero)
  for (int e = tid; e < kQB * kQB; e += kQThreads) {
    const int k = e / kQB, c = e % kQB;
    double a = 0.0;
    for (int g = 0; g < cols; ++g) a = fma(vt[g * P + k], bs[g * P + c], a);
    ws[k * P + c] = a;
  }
  __syncthreads();
  // M = T W (T upper triangular), staged through registers; V rows of the tile
  constexpr int kPer = kQB * kQB / kQThreads;
  double mreg[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = tid + u * kQThreads;
    const int k = e / kQB, c = e % kQB;
    double a = 0.0;
    for (int l = k; l < kQB; ++l) a = fma(tsm[k * P + l], ws[l * P + c], a);
    mreg[u] = a;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = tid + u * kQThreads;
    ws[(e / kQB) * P + (e % kQB)] = mreg[u];
  }
  for (int e = tid; e < kApRows * kQB; e += kQThreads) {
    const int g = e / kQB, k = e % kQB, gl = r0 + g;
    cp_async_f64(&vr[g * P + k], V + (c0 + (g < nr ? gl : 0)) * kQB + k, g < nr);
  }
  cp_async_wait_all();
  __syncthreads();
  if (r0 < kQB && tid < kApRows && r0 + tid < kQB && tid < nr) vr[tid * P + r0 + tid] = 1.0;
  __syncthreads();
  // Out rows = [B; 0] - V M
  for (int e = tid; e < kApRows * kQB; e += kQThreads) {
    const int g = e / kQB, c = e % kQB;
    if (g >= nr || c >= cols) continue;
    const int gl = r0 + g;
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int k = 0; k < kQB; k += 2) {
      a = fma(vr[g * P + k], ws[k * P + c], a);
      b = fma(vr[g * P + k + 1], ws[(k + 1) * P + c], b);
    }
    const double base = gl < kQB ? b_at(gl, c) : 0.0;
    Out[(c0 + gl) * ldo + c] = base - (a + b);
  }
}

// cluster size for a level of `r` rows: one cluster covers up to 16 CTAs
// (4096 rows); 16-CTA clusters are a non-portable size -- fall back to 8
static int g_max_cluster = 0;

static int launch_leaf(int ns, int nch, int cl, const double* in, int64_t r, int cols, int64_t in_ld, double* V,
                       double* T, double* Rs, double* R, int64_t ldr, double* sgn, cudaStream_t s,
                       double* Mg = nullptr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch * cl);
  cfg.blockDim = dim3(kQThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // SPB_PDL_ENTRY in the kernel
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  const cudaError_t e =
      ns == kQSlotsTall ? cudaLaunchKernelEx(&cfg, tsqr_leaf_kernel<kQSlotsTall>, in, r, cols, in_ld, V, T, Rs, R, ldr, sgn, Mg)
                        : cudaLaunchKernelEx(&cfg, tsqr_leaf_kernel<32>, in, r, cols, in_ld, V, T, Rs, R, ldr, sgn, Mg);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("tsqr leaf launch: ") + cudaGetErrorString(e));
    return SP_ECUDA;
  }
  count_launch();
  return SP_OK;
}

static int max_cluster() {
  if (g_max_cluster == 0) {
    int mc = 8;
    if (cudaFuncSetAttribute(tsqr_leaf_kernel<32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
        cudaFuncSetAttribute(tsqr_leaf_kernel<kQSlotsTall>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
            cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(kQMaxCluster);
      cfg.blockDim = dim3(kQThreads);
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = kQMaxCluster;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int nclusters = 0;
      int ntall = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, tsqr_leaf_kernel<32>, &cfg) == cudaSuccess && nclusters > 0 &&
          cudaOccupancyMaxActiveClusters(&ntall, tsqr_leaf_kernel<kQSlotsTall>, &cfg) == cudaSuccess && ntall > 0)
        mc = kQMaxCluster;
    }
    cudaGetLastError();
    g_max_cluster = mc;
  }
  return g_max_cluster;
}

// Factor phase: the leaf tree (R written to R); the Q phase (tsqr_form_q)
// is separate so callers that only need R (the Rayleigh-Ritz core of a
// converged subspace step) skip it.  Workspaces live in `ar`.
int tsqr_factor(int64_t rows, int cols, const double* X, int64_t ldx, double* R, int64_t ldr, TsqrPlan& plan,
                Arena& ar, cudaStream_t s) {
  plan = TsqrPlan();
  plan.cols = cols;
  const double* in = X;
  int64_t in_ld = ldx;
  int64_t r = rows;
  plan.sgn = ar.alloc<double>(kQB);
  if (!plan.sgn) {
    set_error("tsqr workspace allocation failed");
    return SP_ECUDA;
  }
  const int mc = max_cluster();
  while (true) {
    TsqrPlan::Level L;
    L.rows = r;
    // clusters only while all chunks fit in one wave: past ~148 CTAs the
    // per-step cluster exchange costs more than the extra tree level it saves
    // 320-row CTAs when that makes the whole level one cluster (one tree
    // level and two apply launches less: cfg3's 5000-row test blocks)
    L.ch = (r > (int64_t)mc * kQCH && r <= (int64_t)mc * kQSlotsTall * kQWarps) ? kQSlotsTall * kQWarps : kQCH;
    const int64_t ctas = ceil_div(r, L.ch);
    L.cl = ctas <= kNumSMs ? (int)std::min<int64_t>(mc, ctas) : 1;
    L.nch = (int)ceil_div(r, (int64_t)L.cl * L.ch);
    L.V = ar.alloc<double>((size_t)r * kQB);
    L.T = ar.alloc<double>((size_t)L.nch * kQB * kQB);
    L.Rs = ar.alloc<double>((size_t)L.nch * cols * kQB);
    if (!L.V || !L.T || !L.Rs) {
      set_error("tsqr workspace allocation failed");
      return SP_ECUDA;
    }
    const bool root = L.nch == 1;
    if (root && plan.lv.empty()) {
      // single chunk: the root leaf also forms M; Q is one small product per row
      plan.Mg = ar.alloc<double>((size_t)kQB * kQB);
      if (!plan.Mg) {
        set_error("tsqr workspace allocation failed");
        return SP_ECUDA;
      }
      SPB_TRY(launch_leaf(L.ch / kQWarps, 1, L.cl, in, r, cols, in_ld, L.V, L.T, L.Rs, R, ldr, plan.sgn, s, plan.Mg));
      plan.lv.push_back(L);
      return SP_OK;
    }
    SPB_TRY(launch_leaf(L.ch / kQWarps, L.nch, L.cl, in, r, cols, in_ld, L.V, L.T, L.Rs, root ? R : nullptr, ldr,
                        root ? plan.sgn : nullptr, s));
    plan.lv.push_back(L);
    if (root) break;
    in = L.Rs;
    in_ld = kQB;
    r = (int64_t)L.nch * cols;
  }
  return SP_OK;
}

int tsqr_form_q(const TsqrPlan& plan, double* Q, int64_t ldq, Arena& ar, cudaStream_t s) {
  const int cols = plan.cols;
  if (plan.Mg) {
    const TsqrPlan::Level& L = plan.lv[0];
    SPB_CUDA(launch_pdl((tsqr_q_kernel), dim3(ceil_div(L.rows, 64)), dim3(kQThreads), 0, s, (const double*)L.V,
                        (const double*)plan.Mg, (const double*)plan.sgn, L.rows, cols, Q, ldq));
    count_launch();
    SPB_CHECK_LAUNCH();
    return SP_OK;
  }
  const double* bin = nullptr;
  for (int l = (int)plan.lv.size() - 1; l >= 0; --l) {
    const TsqrPlan::Level& L = plan.lv[l];
    double* out;
    int64_t ldo;
    if (l == 0) {
      out = Q;
      ldo = ldq;
    } else {
      out = ar.alloc<double>((size_t)L.rows * kQB);
      if (!out) {
        set_error("tsqr workspace allocation failed");
        return SP_ECUDA;
      }
      ldo = kQB;
    }
    const int chunk_rows = L.cl * L.ch;
    SPB_CUDA(launch_pdl((tsqr_apply_kernel), dim3(L.nch * (chunk_rows / kApRows)), dim3(kQThreads), 0, s,
                        (const double*)L.V, (const double*)L.T, L.rows, cols, chunk_rows, bin,
                        (const double*)plan.sgn, out, ldo));
    count_launch();
    SPB_CHECK_LAUNCH();
    bin = out;
  }
  return SP_OK;
}

static int tsqr32(int64_t rows, int cols, const double* X, int64_t ldx, double* Q, int64_t ldq, double* R,
                  int64_t ldr, cudaStream_t s) {
  Arena ar(s);
  TsqrPlan plan;
  SPB_TRY(tsqr_factor(rows, cols, X, ldx, R, ldr, plan, ar, s));
  return tsqr_form_q(plan, Q, ldq, ar, s);
}

__global__ void copy_block(int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst,
                           int64_t ldd) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t i = e / cols, c = e % cols;
  dst[i * ldd + c] = src[i * lds + c];
}

__global__ void add_block(int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst,
                          int64_t ldd) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t i = e / cols, c = e % cols;
  dst[i * ldd + c] += src[i * lds + c];
}

// Wide inputs: panels, two block Gram-Schmidt passes against the previous
// panels, then a Householder TSQR of the projected panel.  Up to 512 columns
// the panels are 32 wide (the register TSQR); wider inputs use 256-wide
// panels factored recursively the same way, so the projections against the
// previous panels are DMMA GEMMs 256 columns wide instead of 32 (round 1's
// 32-wide panels ran cfg5's 262144 x 2000 at ~13 TF/s plus a split-K reduce
// per product).
int tsqr(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
         double* R, int64_t ldr, cudaStream_t s) {
  SPB_REQUIRE(cols >= 1 && rows >= cols, "tsqr needs rows >= cols >= 1");
  SPB_REQUIRE(ldx >= cols && ldq >= cols && ldr >= cols, "bad tsqr leading dimension");
  if (cols <= kQB) return tsqr32(rows, (int)cols, X, ldx, Q, ldq, R, ldr, s);
  const int pw = cols > 512 ? 256 : kQB;  // panel width
  auto panel_qr = [&](const double* P, int w, double* Qp, double* Rp) -> int {
    return pw == kQB ? tsqr32(rows, w, P, w, Qp, ldq, Rp, ldr, s) : tsqr(rows, w, P, w, Qp, ldq, Rp, ldr, s);
  };
  SPB_CUDA(cudaMemset2DAsync(R, ldr * sizeof(double), 0, cols * sizeof(double), cols, s));
  Arena ar(s);
  SPB_ALLOC(ar, double, P, (size_t)rows * pw);
  SPB_ALLOC(ar, double, T, (size_t)cols * pw);
  SPB_ALLOC(ar, double, S2, (size_t)cols * pw);
  SPB_ALLOC(ar, double, R2, (size_t)pw * pw);
  SPB_ALLOC(ar, double, R3, (size_t)pw * pw);
  for (int64_t p0 = 0; p0 < cols; p0 += pw) {
    const int w = (int)std::min<int64_t>(pw, cols - p0);
    copy_block<<<ceil_div(rows * w, 256), 256, 0, s>>>(rows, w, X + p0, ldx, P, w);
    count_launch();
    SPB_CHECK_LAUNCH();
    if (p0 > 0) {
      for (int pass = 0; pass < 2; ++pass) {
        // T = Q[:, :p0]^T P ; P -= Q[:, :p0] T ; R[:p0, p0:p0+w] += T
        SPB_TRY(gemm(1, 0, p0, w, rows, 1.0, Q, ldq, P, w, 0.0, T, w, s));
        SPB_TRY(gemm(0, 0, rows, w, p0, -1.0, Q, ldq, T, w, 1.0, P, w, s));
        add_block<<<ceil_div(p0 * w, 256), 256, 0, s>>>(p0, w, T, w, R + p0, ldr);
        count_launch();
        SPB_CHECK_LAUNCH();
      }
    }
    double* Qp = Q + p0;
    double* Rp = R + p0 * ldr + p0;
    SPB_TRY(panel_qr(P, w, Qp, Rp));
    if (p0 > 0) {
      // A numerically rank-deficient panel leaves a residual P of rounding
      // size whose components along Q[:, :p0] are as large as the rest, so
      // orth(P) is not orthogonal to the previous panels: re-orthogonalise
      // the NORMALISED panel (twice) and QR it again.
      //   Qp = Q S + Q' R'  ->  R[:p0, panel] += S Rp,  R_panel = R' Rp
      for (int pass = 0; pass < 2; ++pass) {
        double* Sx = pass == 0 ? T : S2;
        SPB_TRY(gemm(1, 0, p0, w, rows, 1.0, Q, ldq, Qp, ldq, 0.0, Sx, w, s));
        SPB_TRY(gemm(0, 0, rows, w, p0, -1.0, Q, ldq, Sx, w, 1.0, Qp, ldq, s));
      }
      add_block<<<ceil_div(p0 * w, 256), 256, 0, s>>>(p0, w, S2, w, T, w);
      count_launch();
      SPB_CHECK_LAUNCH();
      SPB_TRY(gemm(0, 0, p0, w, w, 1.0, T, w, Rp, ldr, 1.0, R + p0, ldr, s));
      copy_block<<<ceil_div(rows * w, 256), 256, 0, s>>>(rows, w, Qp, ldq, P, w);
      count_launch();
      SPB_CHECK_LAUNCH();
      // R2 (w x w, ld w): the panel QR writes R into a (w x w) block with ld ldr
      // in the recursive case, so factor into R2 with its own leading dimension
      if (pw == kQB)
        SPB_TRY(tsqr32(rows, w, P, w, Qp, ldq, R2, w, s));
      else
        SPB_TRY(tsqr(rows, w, P, w, Qp, ldq, R2, w, s));
      SPB_TRY(gemm(0, 0, w, w, w, 1.0, R2, w, Rp, ldr, 0.0, R3, w, s));
      copy_block<<<ceil_div(w * w, 256), 256, 0, s>>>(w, w, R3, w, Rp, ldr);
      count_launch();
      SPB_CHECK_LAUNCH();
    }
  }
  return SP_OK;
}

}  // namespace spb
