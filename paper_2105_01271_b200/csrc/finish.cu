// Fused finish stage of the single-pass pipelines (r <= 16 kept columns).
//
// Given Z = U_r (m x r, the kept left basis of the sketch) and the output of
// the one read of A, Y = A^T Z (n x r), the pipelines return the rank-k SVD
// of P_r A = Z Y^T:
//   Y = Q R (shifted CholeskyQR2),  R^T = Us S Vs^T (one-sided Jacobi),
//   U = [Z Us | completion],  V = [Q Vs | completion]   (rank-k padding,
//   tests/test_svd.py:163-171 of the reference).
// This replaces LAPACK thin_qr / thin_svd / the GEMMs of src/svd.py:168-189
// and src/power.py:158-181 for the kept part.  Launches after the A pass:
//   gram_rows (partial Grams of Y; the last CTA reduces them in a fixed
//     order and factors G1 + s I = R1^T R1, shift s = 16 r eps tr(G1))
//   -> gram_rows (partial Grams of Q1 = Y R1^{-1}, Q1 never stored)
//   -> finish_core (1 CTA: Cholesky of Q1^T Q1 -> R2, R = R2 R1, Jacobi SVD
//      of R^T, the top k rows of both factors and both Householder
//      completions, concurrently in two thread groups)
//   -> finish_rows (one streaming pass writing U and V).
// No host synchronisation: the diagonal shift makes the first Cholesky
// unconditionally defined and the second pass restores O(eps) orthogonality
// for kappa(Y) up to ~1e7 (the caller routes kappa >= 1e6 to Householder
// TSQR).  A non-positive or non-finite pivot (non-finite A) raises a device
// flag the host reads lazily (sp_deferred_status), and S is poisoned with NaN.
// Every reduction runs in a fixed order: bitwise reproducible.
#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

constexpr int kFcMaxR = 16;
constexpr int kMR = kFcMaxR;
constexpr double kFcJacTol = 1e-15;  // jacobi.cu kJacTol
constexpr int kFcMaxSweeps = 40;
typedef double SmallMat[kMR][kMR + 1];

struct JacSmem {
  double sig[32];
  signed char ptab[31][32];
  int act[32], pos[32];
  int na;
};

// circle-method partner of position x among na (even) players in round r
__device__ __forceinline__ int fc_partner(int x, int r, int na) {
  const int n1 = na - 1;
  if (x == 0) return 1 + (r % n1);
  int y = (2 * r - (x - 1)) % n1;
  if (y < 0) y += n1;
  y += 1;
  return y == x ? 0 : y;
}

// One warp: one-sided Jacobi on M (r x r, r <= RPW), lane c holding column c
// (x[i] = M[i][c]); rotations accumulated in v.  Same rotation formula,
// threshold and negligible-column rule as jacobi32_kernel (jacobi.cu).
template <int RPW>
__device__ void fc_jacobi_warp(int r, double (&x)[RPW], double (&v)[RPW], JacSmem& sh, int c) {
  double a0 = 0.0;
#pragma unroll
  for (int k = 0; k < RPW; ++k) a0 = fma(x[k], x[k], a0);
  // ||M||_F^2 in lane order (identical in every lane)
  sh.sig[c] = a0;
  __syncwarp();
  double fro = 0.0;
  for (int cc = 0; cc < 32; ++cc) fro += sh.sig[cc];
  const double negl = 1e-30 * fro;
  if (c == 0) {
    int na = 0;
    for (int cc = 0; cc < 32; ++cc) sh.pos[cc] = -1;
    for (int cc = 0; cc < r; ++cc)
      if (sh.sig[cc] > negl) {
        sh.pos[cc] = na;
        sh.act[na++] = cc;
      }
    if (na & 1) sh.act[na++] = -1;
    sh.na = na;
  }
  __syncwarp();
  const int na = sh.na;
  for (int rd = 0; rd < na - 1; ++rd) {
    const int ps = sh.pos[c];
    sh.ptab[rd][c] = (signed char)(ps >= 0 ? sh.act[fc_partner(ps, rd, na)] : -1);
  }
  __syncwarp();
  for (int sweep = 0; sweep < kFcMaxSweeps && na >= 2; ++sweep) {
    int rotated = 0;
    for (int round = 0; round < na - 1; ++round) {
      const int plane = sh.ptab[round][c];
      const int src = plane >= 0 ? plane : c;
      double y[RPW], z[RPW];
#pragma unroll
      for (int k = 0; k < RPW; ++k) {
        y[k] = __shfl_sync(0xffffffffu, x[k], src);
        z[k] = __shfl_sync(0xffffffffu, v[k], src);
      }
      double pa0 = x[0] * x[0], pa1 = x[1] * x[1], pg0 = x[0] * y[0], pg1 = x[1] * y[1];
#pragma unroll
      for (int k = 2; k < RPW; k += 2) {
        pa0 = fma(x[k], x[k], pa0);
        pa1 = fma(x[k + 1], x[k + 1], pa1);
        pg0 = fma(x[k], y[k], pg0);
        pg1 = fma(x[k + 1], y[k + 1], pg1);
      }
      const double a = pa0 + pa1, g = pg0 + pg1;
      const double b = __shfl_sync(0xffffffffu, a, src);
      if (plane < 0) continue;
      const bool low = c < plane;
      const double ap = low ? a : b, aq = low ? b : a;
      const double apq = ap * aq;
      const bool big = !(apq < 1e300);
      if (!(g != 0.0 && fmin(ap, aq) > negl &&
            (big ? fabs(g) > kFcJacTol * sqrt(ap) * sqrt(aq) : g * g > (kFcJacTol * kFcJacTol) * apq)))
        continue;
      const double d = aq - ap, h = 2.0 * g;
      const double ad = fabs(d), ah = fabs(h);
      double cs, sn;
      if (ad < 1e140 && ah < 1e140 && (ad > 1e-140 || ah > 1e-140)) {
        // fast path, two dependent MUFU rsqrt (+ Newton) stages: rh =
        // 1 / hypot(d, h) gives cos 2theta = |d| rh and sin 2theta = h rh
        // (|theta| <= pi / 4); cs = sqrt((1 + cos 2theta) / 2) and
        // sn = sin 2theta / (2 cs) share one rsqrt of u in [1/2, 1]
        const double s2 = fma(d, d, h * h);
        const double rh = fast_rsqrt(s2);
        const double u = fma(0.5 * ad, rh, 0.5);
        const double w = fast_rsqrt(u);
        cs = u * w;
        sn = (copysign(0.5, d) * h) * (rh * w);
      } else {
        const double t = copysign(1.0, d) * h / (ad + hypot(d, h));
        cs = rsqrt(fma(t, t, 1.0));
        sn = cs * t;
      }
      const double so = low ? -sn : sn;
#pragma unroll
      for (int k = 0; k < RPW; ++k) {
        x[k] = fma(so, y[k], cs * x[k]);
        v[k] = fma(so, z[k], cs * v[k]);
      }
      rotated = 1;
    }
    if (!__any_sync(0xffffffffu, rotated)) break;
  }
}

// Cholesky of the c x c SPD matrix G (c <= 16, smem) by ONE warp, in place:
// G -> R (upper, R^T R = G + shift_rel tr(G) I), Ri = R^{-1}.  Pivots by
// rsqrt (no division); false (uniform) on a non-positive / non-finite pivot.
template <int R>
__device__ bool chol_inv_warp(SmallMat& G, SmallMat& Ri, double* rdiag, double shift_rel, int lane) {
  constexpr int c = R;
  if (shift_rel > 0.0) {
    double tr = 0.0;
    for (int i = 0; i < c; ++i) tr += G[i][i];
    __syncwarp();
    if (lane < c) G[lane][lane] += shift_rel * tr;
    __syncwarp();
  }
  for (int j = 0; j < c; ++j) {
    const double d = G[j][j];
    if (!(d > 0.0) || !(d < INFINITY)) return false;
    const double rs = fast_range(d) ? fast_rsqrt(d) : rsqrt(d);
    __syncwarp();
    if (lane >= j && lane < c) G[j][lane] = lane == j ? d * rs : G[j][lane] * rs;
    if (lane == j) rdiag[j] = rs;
    __syncwarp();
    const int w = c - j - 1;
    for (int e = lane; e < w * w; e += 32) {
      const int i = j + 1 + e / w, l = j + 1 + e % w;
      if (l >= i) G[i][l] = fma(-G[j][i], G[j][l], G[i][l]);
    }
    __syncwarp();
  }
  // column l of R^{-1} by back substitution, lane l, in registers
  if (lane < c) {
    double riv[R];
#pragma unroll
    for (int i = R - 1; i >= 0; --i) {
      double acc = (i == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int q = i + 1; q < R; ++q)
        if (q <= lane) acc = fma(-G[i][q], riv[q], acc);
      riv[i] = (i <= lane && i < c) ? acc * rdiag[i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (i < c) Ri[i][lane] = riv[i];
  }
  for (int e = lane; e < c * c; e += 32)
    if (e % c < e / c) G[e / c][e % c] = 0.0;  // clear the strict lower part
  __syncwarp();
  return true;
}

// ------------------------------------------------------------- Gram pass ----
// partial[cta] = sum over the CTA's rows of x x^T (r x r), x = Y row, or
// (Q1) x = y R1^{-1} in a fixed summation order shared with finish_core and
// finish_rows.  With `tail`, the last CTA to finish (atomic ticket) sums the
// partials in CTA order and factors them: R1, R1^{-1} (shifted Cholesky).
constexpr int kGrThreads = 256;
constexpr int kGrChunk = 256;  // rows staged per step

struct GramTail {
  int* ticket;       // zero on entry, reset to zero by the last CTA
  double* R;         // r x r out (upper)
  double* Rinv;      // r x r out
  int* flag;         // OR-ed on breakdown
  double shift_rel;
};

template <int R>
__global__ void __launch_bounds__(kGrThreads)
gram_rows_kernel(int64_t rows, const double* __restrict__ Y, const double* __restrict__ R1i,
                 int64_t rows_per_cta, double* __restrict__ partial, GramTail tail) {
  SPB_PDL_ENTRY();
  constexpr int r = R;
  __shared__ __align__(16) double ys[kGrChunk * R];
  __shared__ SmallMat ri, G, Ri;
  __shared__ double red[kGrThreads], rdiag[kMR];
  __shared__ int last;
  const int tid = threadIdx.x, nout = r * r;
  const int ng = kGrThreads / nout;  // row groups
  const int o = tid % nout, rg = tid / nout;
  const int a = o / r, b = o % r;
  if (R1i)
    for (int e = tid; e < nout; e += kGrThreads) ri[e / r][e % r] = R1i[e];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = imin64(rows, r0 + rows_per_cta);
  double acc0 = 0.0, acc1 = 0.0;
  for (int64_t c0 = r0; c0 < r1; c0 += kGrChunk) {
    const int nr = (int)imin64(kGrChunk, r1 - c0);
    for (int e = tid; e < nr * r; e += kGrThreads) cp_async_f64(&ys[e], Y + c0 * r + e, true);
    cp_async_wait_all();
    __syncthreads();
    if (R1i && tid < nr) {  // x = y R1^{-1} in place (thread per row)
      double x[R], q[R];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        x[i] = i < r ? ys[tid * r + i] : 0.0;
        q[i] = 0.0;
      }
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (i < r) {
#pragma unroll
          for (int j = 0; j < R; ++j)
            if (j < r) q[j] = fma(x[i], ri[i][j], q[j]);
        }
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (j < r) ys[tid * r + j] = q[j];
    }
    __syncthreads();
    if (rg < ng) {
      int i = rg;
      for (; i + ng < nr; i += 2 * ng) {
        acc0 = fma(ys[i * r + a], ys[i * r + b], acc0);
        acc1 = fma(ys[(i + ng) * r + a], ys[(i + ng) * r + b], acc1);
      }
      if (i < nr) acc0 = fma(ys[i * r + a], ys[i * r + b], acc0);
    }
    __syncthreads();
  }
  red[tid] = rg < ng ? acc0 + acc1 : 0.0;
  __syncthreads();
  if (tid < nout) {
    double t = 0.0;
    for (int g = 0; g < ng; ++g) t += red[g * nout + tid];
    partial[(int64_t)blockIdx.x * nout + tid] = t;
  }
  if (!tail.ticket) return;
  // ---- last CTA: fixed-order reduction of the partials and the factorisation
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(tail.ticket, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  {
    const int nb = gridDim.x;
    double s0 = 0.0, s1 = 0.0;
    if (rg < ng) {
      int bb = rg;
      for (; bb + ng < nb; bb += 2 * ng) {
        s0 += __ldcg(partial + (int64_t)bb * nout + o);
        s1 += __ldcg(partial + (int64_t)(bb + ng) * nout + o);
      }
      if (bb < nb) s0 += __ldcg(partial + (int64_t)bb * nout + o);
    }
    red[tid] = rg < ng ? s0 + s1 : 0.0;
    __syncthreads();
    if (tid < nout) {
      double t = 0.0;
      for (int g = 0; g < ng; ++g) t += red[g * nout + tid];
      G[tid / r][tid % r] = t;
    }
    __syncthreads();
  }
  if (tid < 32) {
    const bool ok = chol_inv_warp<R>(G, Ri, rdiag, tail.shift_rel, tid);
    if (!ok) {
      if (tid == 0) atomicOr(tail.flag, 1);
    }
    for (int e = tid; e < nout; e += 32) {
      tail.R[e] = ok ? G[e / r][e % r] : 0.0;
      tail.Rinv[e] = ok ? Ri[e / r][e % r] : 0.0;
    }
    if (tid == 0) *tail.ticket = 0;
  }
}

// Streaming variant for R <= 8 (every BASELINE configuration): thread per
// row, the R (R + 1) / 2 products accumulated in registers, no shared-memory
// staging or per-chunk barriers -- a plain read of Y at HBM rate even when n
// is 10^6..10^7 (the staged kernel above is latency-bound there).  Same tail.
constexpr int kGsThreads = 256;

template <int R>
__global__ void __launch_bounds__(kGsThreads)
gram_stream_kernel(int64_t rows, const double* __restrict__ Y, const double* __restrict__ R1i,
                   double* __restrict__ partial, GramTail tail) {
  SPB_PDL_ENTRY();
  constexpr int NP = R * (R + 1) / 2, nout = R * R;
  __shared__ double ri[R][R];
  __shared__ double red[kGsThreads / 32][NP];
  __shared__ SmallMat G, Ri;
  __shared__ double rdiag[kMR];
  __shared__ int last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (R1i)
    for (int e = tid; e < nout; e += kGsThreads) ri[e / R][e % R] = R1i[e];
  __syncthreads();
  double acc[NP];
#pragma unroll
  for (int e = 0; e < NP; ++e) acc[e] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kGsThreads;
  for (int64_t row = (int64_t)blockIdx.x * kGsThreads + tid; row < rows; row += stride) {
    double x[R];
    const double* yr = Y + row * R;
#pragma unroll
    for (int i = 0; i < R; ++i) x[i] = __ldg(yr + i);
    if (R1i) {  // x = y R1^{-1}, the summation order of gram_rows / finish_core / finish_rows
      double q[R];
#pragma unroll
      for (int j = 0; j < R; ++j) q[j] = 0.0;
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j = 0; j < R; ++j) q[j] = fma(x[i], ri[i][j], q[j]);
#pragma unroll
      for (int j = 0; j < R; ++j) x[j] = q[j];
    }
    int e = 0;
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = a; b < R; ++b) {
        acc[e] = fma(x[a], x[b], acc[e]);
        ++e;
      }
  }
  // warp sums (fixed shuffle order), then the 8 warps in order
#pragma unroll
  for (int e = 0; e < NP; ++e) {
    const double v = warp_sum(acc[e]);
    if (lane == 0) red[warp][e] = v;
  }
  __syncthreads();
  if (tid < nout) {
    const int a = tid / R, b = tid % R;
    const int e = a <= b ? a * R - a * (a - 1) / 2 + (b - a) : b * R - b * (b - 1) / 2 + (a - b);
    double t = 0.0;
    for (int w = 0; w < kGsThreads / 32; ++w) t += red[w][e];
    partial[(int64_t)blockIdx.x * nout + tid] = t;
  }
  if (!tail.ticket) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(tail.ticket, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  {
    // all threads: gs groups of nout, group g sums partials g, g + gs, ...
    // (two chains), then the group sums in group order -- a fixed order
    constexpr int gs = kGsThreads / nout;
    __shared__ double gred[gs * nout];
    const int o = tid % nout, g = tid / nout;
    const int nb = gridDim.x;
    double s0 = 0.0, s1 = 0.0;
    if (g < gs) {
      int bb = g;
      for (; bb + gs < nb; bb += 2 * gs) {
        s0 += __ldcg(partial + (int64_t)bb * nout + o);
        s1 += __ldcg(partial + (int64_t)(bb + gs) * nout + o);
      }
      if (bb < nb) s0 += __ldcg(partial + (int64_t)bb * nout + o);
      gred[g * nout + o] = s0 + s1;
    }
    __syncthreads();
    if (tid < nout) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < gs; ++q) t += gred[q * nout + tid];
      G[tid / R][tid % R] = t;
    }
  }
  __syncthreads();
  if (tid < 32) {
    const bool ok = chol_inv_warp<R>(G, Ri, rdiag, tail.shift_rel, tid);
    if (!ok && tid == 0) atomicOr(tail.flag, 1);
    for (int e = tid; e < nout; e += 32) {
      tail.R[e] = ok ? G[e / R][e % R] : 0.0;
      tail.Rinv[e] = ok ? Ri[e / R][e % R] : 0.0;
    }
    if (tid == 0) *tail.ticket = 0;
  }
}

// ------------------------------------------------------------ the core ----
// Householder-reconstruction completion (complete.cu header) of the r x k
// problem X (k x r top rows of an orthonormal N x r factor, smem) for the
// product factor B (r x r): writes Mf = [B | -B K'] (r x k) and
// Etf = [0 | E'] (k x k) to global.  Run by a 256-thread group; both groups of
// the CTA execute the same barrier sequence (same r, k).
struct HcSmall {
  SmallMat W, Ui, Li, T, Lp, G, BG;
  double S[kMR], rd[kMR];
};

template <int R>
__device__ void hh_small(int k, const double* __restrict__ X, const SmallMat& B, HcSmall& h,
                         double* __restrict__ Mf, double* __restrict__ Etf, int t) {
  constexpr int r = R, nout = R * R;
  if (t < 32) {
    // LU without pivoting of X[0:r, 0:r] - S, S_i = -sign(pivot): |pivot| >= 1
    for (int e = t; e < nout; e += 32) h.W[e / r][e % r] = X[e];
    __syncwarp();
    for (int i = 0; i < r; ++i) {
      const double w = h.W[i][i];
      const double s = w >= 0.0 ? -1.0 : 1.0;
      const double piv = w - s;
      const double rp = fast_range(fabs(piv)) ? fast_rcp(piv) : 1.0 / piv;  // |piv| >= 1
      __syncwarp();
      if (t == 0) {
        h.S[i] = s;
        h.W[i][i] = piv;
        h.rd[i] = rp;
      }
      if (t > i && t < r) h.W[t][i] *= rp;  // L multipliers
      __syncwarp();
      const int w2 = r - i - 1;
      for (int e = t; e < w2 * w2; e += 32) {
        const int a = i + 1 + e / w2, b = i + 1 + e % w2;
        h.W[a][b] = fma(-h.W[a][i], h.W[i][b], h.W[a][b]);
      }
      __syncwarp();
    }
    // lanes 0..r-1: column of U^{-1}; lanes 16..16+r-1: column of L1^{-1}
    if (t < r) {
      const int col = t;
      double u[R];
#pragma unroll
      for (int a = R - 1; a >= 0; --a) {
        double acc = (a == col) ? 1.0 : 0.0;
#pragma unroll
        for (int b = a + 1; b < R; ++b)
          if (b <= col) acc = fma(-h.W[a][b], u[b], acc);
        u[a] = (a <= col && a < r) ? acc * h.rd[a] : 0.0;
      }
#pragma unroll
      for (int a = 0; a < R; ++a)
        if (a < r) h.Ui[a][col] = u[a];
    } else if (t >= 16 && t < 16 + r) {
      const int col = t - 16;
      double l[R];
#pragma unroll
      for (int a = 0; a < R; ++a) {
        double acc = (a == col) ? 1.0 : 0.0;
#pragma unroll
        for (int b = 0; b < R; ++b)
          if (b < a && b >= col) acc = fma(-h.W[a][b], l[b], acc);
        l[a] = (a >= col && a < r) ? acc : 0.0;
      }
#pragma unroll
      for (int a = 0; a < R; ++a)
        if (a < r) h.Li[a][col] = l[a];
    }
  }
  __syncthreads();
  const int a = t / r, b = t % r;
  const bool act = t < nout;
  if (act) {  // T = -U S L1^{-T}
    double acc = 0.0;
    for (int q = a; q < r; ++q) acc = fma(h.W[a][q] * h.S[q], h.Li[b][q], acc);
    h.T[a][b] = -acc;
  }
  __syncthreads();
  if (act) {  // Lp = T U^{-T}
    double acc = 0.0;
    for (int q = b; q < r; ++q) acc = fma(h.T[a][q], h.Ui[b][q], acc);
    h.Lp[a][b] = acc;
  }
  __syncthreads();
  if (act) {  // G = U^{-1} Lp
    double acc = 0.0;
    for (int q = a; q < r; ++q) acc = fma(h.Ui[a][q], h.Lp[q][b], acc);
    h.G[a][b] = acc;
  }
  __syncthreads();
  if (act) {  // BG = B G
    double acc = 0.0;
    for (int q = 0; q < r; ++q) acc = fma(B[a][q], h.G[q][b], acc);
    h.BG[a][b] = acc;
  }
  __syncthreads();
  // Mf[i][j] = B[i][j] (j < r), -sum_p BG[i][p] X[j][p] (j >= r)
  for (int e = t; e < r * k; e += 256) {
    const int i = e / k, j = e % k;
    double v;
    if (j < r) {
      v = B[i][j];
    } else {
      double acc = 0.0;
#pragma unroll
      for (int p = 0; p < R; ++p)
        if (p < r) acc = fma(h.BG[i][p], X[j * r + p], acc);
      v = -acc;
    }
    Mf[e] = v;
  }
  // Etf[i][j] = 0 (j < r); S_i sum_p G[i][p] X[j][p] (i < r <= j); I (i, j >= r)
  for (int e = t; e < k * k; e += 256) {
    const int i = e / k, j = e % k;
    double v = 0.0;
    if (j >= r) {
      if (i < r) {
        double acc = 0.0;
#pragma unroll
        for (int p = 0; p < R; ++p)
          if (p < r) acc = fma(h.G[i][p], X[j * r + p], acc);
        v = h.S[i] * acc;
      } else {
        v = (i == j) ? 1.0 : 0.0;
      }
    }
    Etf[e] = v;
  }
}

constexpr int kFcThreads = 512;

struct FcShared {
  HcSmall hc[2];
  SmallMat G, R2i, R1, R1i, R, Us, Vs, Bv;
  JacSmem jac;
  double red[kFcThreads];
  double rdiag[kMR];
  int bad;
  // followed by Zt, Yt (k x r), XU, XV (k x r)
};

// S (k): sigma desc, zero padded; MfU / MfV (r x k), EtfU / EtfV (k x k):
// U = Z MfU + [EtfU; 0],  V = (Y R1^{-1}) MfV + [EtfV; 0].
template <int R>
__global__ void __launch_bounds__(kFcThreads)
finish_core_kernel(int k, int nb2, const double* __restrict__ P2, const double* __restrict__ R1g,
                   const double* __restrict__ R1ig, const double* __restrict__ Z, int64_t ldz,
                   const double* __restrict__ Y, int64_t ldy, double* __restrict__ S,
                   double* __restrict__ MfU, double* __restrict__ EtfU, double* __restrict__ MfV,
                   double* __restrict__ EtfV, int* flag, int* hflag) {
  SPB_PDL_ENTRY();
  extern __shared__ __align__(16) unsigned char fc_smem[];
  FcShared& sh = *reinterpret_cast<FcShared*>(fc_smem);
  double* Zt = reinterpret_cast<double*>(fc_smem + (sizeof(FcShared) + 15) / 16 * 16);
  constexpr int r = R, nout = R * R, RPW = R < 2 ? 2 : R + (R & 1);
  double* Yt = Zt + k * r;
  double* XU = Yt + k * r;
  double* XV = XU + k * r;
  const int tid = threadIdx.x;
  SPB_TDECL;
  SPB_TMARK(0);
  if (tid == 0) sh.bad = 0;
  for (int e = tid; e < nout; e += kFcThreads) {
    cp_async_f64(&sh.R1[e / r][e % r], R1g + e, true);
    cp_async_f64(&sh.R1i[e / r][e % r], R1ig + e, true);
  }
  for (int e = tid; e < k * r; e += kFcThreads) {
    const int i = e / r, l = e % r;
    cp_async_f64(&Zt[e], Z + (int64_t)i * ldz + l, true);
    cp_async_f64(&Yt[e], Y + (int64_t)i * ldy + l, true);
  }
  // (a) fixed-order reduction of the nb2 partial Grams of Q1 (loads in flight)
  {
    const int gs = kFcThreads / nout;
    const int o = tid % nout, g = tid / nout;
    double a0 = 0.0, a1 = 0.0;
    if (g < gs) {
      int b = g;
      for (; b + gs < nb2; b += 2 * gs) {
        a0 += P2[(int64_t)b * nout + o];
        a1 += P2[(int64_t)(b + gs) * nout + o];
      }
      if (b < nb2) a0 += P2[(int64_t)b * nout + o];
    }
    sh.red[tid] = g < gs ? a0 + a1 : 0.0;
    cp_async_wait_all();
    __syncthreads();
    if (tid < nout) {
      double t = 0.0;
      for (int q = 0; q < gs; ++q) t += sh.red[q * nout + tid];
      sh.G[tid / r][tid % r] = t;
    }
    __syncthreads();
  }
  SPB_TMARK(1);
  // (b) warp 0: R2 (Cholesky of Q1^T Q1), R = R2 R1, Jacobi SVD of R^T
  if (tid < 32) {
    const int lane = tid;
    const bool ok = chol_inv_warp<R>(sh.G, sh.R2i, sh.rdiag, 0.0, lane);
    if (!ok) {
      if (lane == 0) sh.bad = 1;
    } else {
      for (int e = lane; e < nout; e += 32) {
        const int i = e / r, l = e % r;
        double acc = 0.0;
        for (int q = i; q <= l; ++q) acc = fma(sh.G[i][q], sh.R1[q][l], acc);
        sh.R[i][l] = (l >= i) ? acc : 0.0;
      }
      __syncwarp();
      SPB_TMARK(2);
      // M = R^T: lane c holds column c of M = row c of R
      double x[RPW], v[RPW];
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        x[i] = (i < r && lane < r) ? sh.R[lane][i] : 0.0;
        v[i] = (i == lane) ? 1.0 : 0.0;
      }
      fc_jacobi_warp<RPW>(r, x, v, sh.jac, lane);
      SPB_TMARK(3);
      double a1 = 0.0;
#pragma unroll
      for (int i = 0; i < RPW; ++i) a1 = fma(x[i], x[i], a1);
      const double sc = sqrt(a1);
      __syncwarp();
      sh.jac.sig[lane] = lane < r ? sc : -1.0;
      __syncwarp();
      int rank = 0;
      for (int d = 0; d < 32; ++d) {
        const double sd = sh.jac.sig[d];
        rank += (sd > sc || (sd == sc && d < lane)) ? 1 : 0;
      }
      if (lane < r) {
        S[rank] = sc;
        const double inv = sc > 0.0 ? 1.0 / sc : 0.0;
#pragma unroll
        for (int i = 0; i < RPW; ++i)
          if (i < r) {
            sh.Us[i][rank] = x[i] * inv;
            sh.Vs[i][rank] = v[i];
          }
      }
      for (int j = r + lane; j < k; j += 32) S[j] = 0.0;
    }
  }
  __syncthreads();
  // The call's status word: the last writer of `flag` publishes it to mapped
  // pinned host memory (read by sp_deferred_status after the caller's sync)
  // and rezeroes it for the next call -- no copy or memset node in the chain
  if (sh.bad) {
    if (tid == 0) {
      atomicExch(flag, 0);
      if (hflag) *(volatile int*)hflag = 1;
      __threadfence_system();
    }
    for (int j = tid; j < k; j += kFcThreads) S[j] = __longlong_as_double(0x7ff8000000000000ll);
    return;  // uniform
  }
  if (tid == 0) {
    const int f = atomicExch(flag, 0);
    if (hflag) *(volatile int*)hflag = f;
    __threadfence_system();
  }
  SPB_TMARK(4);
  // (c) Bv = R2^{-1} Vs; Q1 top rows = Yt R1^{-1} (in place); XU = Zt Us
  if (tid < nout) {
    const int i = tid / r, l = tid % r;
    double acc = 0.0;
    for (int q = i; q < r; ++q) acc = fma(sh.R2i[i][q], sh.Vs[q][l], acc);
    sh.Bv[i][l] = acc;
  }
  for (int e = tid; e < k * r; e += kFcThreads) {
    const int i = e / r, l = e % r;
    double au = 0.0, q1 = 0.0;
#pragma unroll
    for (int p = 0; p < R; ++p)
      if (p < r) {
        au = fma(Zt[i * r + p], sh.Us[p][l], au);
        q1 = fma(Yt[i * r + p], sh.R1i[p][l], q1);  // x = y R1^{-1}, gram_rows' order
      }
    XU[e] = au;
    XV[e] = q1;  // parked; XV = Q1top Bv below
  }
  __syncthreads();
  {
    // XV = Q1top Bv (Q1top parked in XV, copy through registers)
    double qv[(R * 256 + kFcThreads - 1) / kFcThreads];
    int cnt = 0;
    for (int e = tid; e < k * r; e += kFcThreads, ++cnt) {
      const int i = e / r, l = e % r;
      double acc = 0.0;
#pragma unroll
      for (int p = 0; p < R; ++p)
        if (p < r) acc = fma(XV[i * r + p], sh.Bv[p][l], acc);
      qv[cnt] = acc;
    }
    __syncthreads();
    cnt = 0;
    for (int e = tid; e < k * r; e += kFcThreads, ++cnt) XV[e] = qv[cnt];
  }
  __syncthreads();
  SPB_TMARK(5);
  // (d) both completions at once: threads [0, 256) -> U, [256, 512) -> V
  const int grp = tid >> 8;
  hh_small<R>(k, grp ? XV : XU, grp ? sh.Bv : sh.Us, sh.hc[grp], grp ? MfV : MfU, grp ? EtfV : EtfU, tid & 255);
  SPB_TMARK(6);
  if (tid == 0) SPB_TPRINT("finish_core reduce/chol/jacobi/sort/xtop/hh", 7);
}

// One streaming pass: rows [0, m) of U (tiles [0, bu)) and [0, n) of V.
// Persistent CTAs walk 128-row tiles; the next tile's input rows are
// prefetched (cp.async, double buffer) while the current one is written.
// Per tile: threads 0..127 form the row inputs (for V, q1 = y R1^{-1} in the
// Gram passes' summation order) into shared memory; then groups of k (warp-
// rounded) threads write whole rows, the threads across the output columns
// (coalesced stores), each thread's Mf column in registers.
constexpr int kFrRows = 128;
constexpr int kFrThreads = 256;

template <int R>
__device__ __forceinline__ void fr_prefetch(int64_t tile, int bu, int64_t m, int64_t n, const double* Z, int64_t ldz,
                                            const double* Y, int64_t ldy, double* buf, int t) {
  const bool isv = tile >= bu;
  const int64_t rows = isv ? n : m;
  const int64_t base = (isv ? tile - bu : tile) * kFrRows;
  const double* X = isv ? Y : Z;
  const int64_t ldx = isv ? ldy : ldz;
  const int nr = (int)imin64(kFrRows, rows - base);
  for (int e = t; e < kFrRows * R; e += kFrThreads) {
    const int rl = e / R, i = e - rl * R;
    const bool ok = rl < nr;
    cp_async_f64(&buf[e], ok ? X + (base + rl) * ldx + i : X, ok);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <int R>
__global__ void __launch_bounds__(kFrThreads)
finish_rows_kernel(int k, int64_t m, int64_t n, int bu, const double* __restrict__ Z, int64_t ldz,
                   const double* __restrict__ Y, int64_t ldy, const double* __restrict__ R1i,
                   const double* __restrict__ MfU, const double* __restrict__ EtfU, const double* __restrict__ MfV,
                   const double* __restrict__ EtfV, double* __restrict__ U, double* __restrict__ V) {
  SPB_PDL_ENTRY();
  extern __shared__ __align__(16) double fr_smem[];
  double* mfu = fr_smem;                   // R x k
  double* mfv = mfu + R * k;               // R x k
  double* ri = mfv + R * k;                // R x R
  double* xb = ri + R * R;                 // 2 x kFrRows x R (input rows, double buffer)
  double* qs = xb + 2 * kFrRows * R;       // kFrRows x (R + 1)
  const int t = threadIdx.x;
  const int64_t ntiles = (int64_t)bu + (n + kFrRows - 1) / kFrRows;
  int64_t tile = blockIdx.x;
  if (tile >= ntiles) return;
  fr_prefetch<R>(tile, bu, m, n, Z, ldz, Y, ldy, xb, t);
  for (int e = t; e < R * k; e += kFrThreads) {
    mfu[e] = MfU[e];
    mfv[e] = MfV[e];
  }
  for (int e = t; e < R * R; e += kFrThreads) ri[e] = R1i[e];
  // column mapping: groups of kh = ceil(k / 2) threads, each thread two
  // adjacent columns (one 16-byte store per row when k is even and the
  // outputs are 16-byte aligned); the ngrp groups take every ngrp-th row of a
  // tile.  Groups are not warp-rounded: a warp's stores then cover the end of
  // one row and the start of the next, still two contiguous segments.
  const int kh = (k + 1) / 2;
  const int ngrp = kFrThreads / kh, grp = t / kh, cl = t - grp * kh;
  const bool vec = (k % 2 == 0) && ((reinterpret_cast<uintptr_t>(U) | reinterpret_cast<uintptr_t>(V)) & 15) == 0;
  for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
    const bool isv = tile >= bu;
    const int64_t rows = isv ? n : m;
    const int64_t base = (isv ? tile - bu : tile) * kFrRows;
    const int nr = (int)imin64(kFrRows, rows - base);
    const double* Et = isv ? EtfV : EtfU;
    double* O = isv ? V : U;
    double* cb = xb + (it & 1) * kFrRows * R;
    // prefetch the next tile into the other buffer, then wait for this one
    const int64_t nxt = tile + gridDim.x;
    if (nxt < ntiles) {
      fr_prefetch<R>(nxt, bu, m, n, Z, ldz, Y, ldy, xb + ((it + 1) & 1) * kFrRows * R, t);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    if (t < nr) {
      double x[R];
#pragma unroll
      for (int i = 0; i < R; ++i) x[i] = cb[t * R + i];
      if (isv) {  // q1 = y R1^{-1}, the Gram passes' summation order
        double q[R];
#pragma unroll
        for (int j = 0; j < R; ++j) q[j] = 0.0;
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
          for (int j = 0; j < R; ++j) q[j] = fma(x[i], ri[i * R + j], q[j]);
#pragma unroll
        for (int j = 0; j < R; ++j) x[j] = q[j];
      }
#pragma unroll
      for (int j = 0; j < R; ++j) qs[t * (R + 1) + j] = x[j];
    }
    __syncthreads();
    const double* mf = isv ? mfv : mfu;
    // thread (group, column pair): the columns' Mf entries in registers, the
    // rows of the tile split over the groups
    if (grp < ngrp) {
      const int c = 2 * cl;
      const bool has1 = c + 1 < k;
      double m0[R], m1[R];
#pragma unroll
      for (int p = 0; p < R; ++p) {
        m0[p] = mf[p * k + c];
        m1[p] = has1 ? mf[p * k + c + 1] : 0.0;
      }
      for (int rl = grp; rl < nr; rl += ngrp) {
        double o0 = 0.0, o1 = 0.0;
#pragma unroll
        for (int p = 0; p < R; ++p) {
          const double q = qs[rl * (R + 1) + p];
          o0 = fma(q, m0[p], o0);
          o1 = fma(q, m1[p], o1);
        }
        const int64_t row = base + rl;
        if (row < k) {
          o0 += Et[row * k + c];
          if (has1) o1 += Et[row * k + c + 1];
        }
        double* dst = O + row * k + c;
        if (vec) {
          *reinterpret_cast<double2*>(dst) = make_double2(o0, o1);
        } else {
          dst[0] = o0;
          if (has1) dst[1] = o1;
        }
      }
    }
    __syncthreads();  // qs and this buffer are rewritten next iteration
  }
}

bool finish_fused_ok(int64_t m, int64_t n, int r, int k) {
  return r >= 1 && r <= kFcMaxR && k >= r && k <= 256 && r * k <= 64 * 64 && m >= k && n >= k && n >= 256;
}

// Y (n x r, ld r) = A^T Z is in place; writes U (m x k), S (k), V (n x k).
// dflag: device int[2] = {flag, ticket}, zeroed by the caller; the flag is
// OR-ed on a Cholesky breakdown / non-finite input.
template <int R>
static int finish_fused_r(int64_t m, int64_t n, const double* Z, int64_t ldz, const double* Y, int k, double* U,
                          double* S, double* V, int* dflag, int* hflag, cudaStream_t s) {
  Arena ar(s);
  // staged Gram kernel: one CTA per SM; streaming kernel (R <= 8): up to 4 per SM
  const bool stream_gram = R <= 8;
  const int nb = stream_gram ? (int)std::min<int64_t>(4 * kNumSMs, ceil_div(n, kGsThreads))
                             : (int)std::min<int64_t>(kNumSMs, ceil_div(n, 64));
  const int64_t rpc = ceil_div(n, nb);
  SPB_ALLOC(ar, double, P1, (size_t)nb * R * R);
  SPB_ALLOC(ar, double, P2, (size_t)nb * R * R);
  SPB_ALLOC(ar, double, R1, (size_t)R * R);
  SPB_ALLOC(ar, double, R1i, (size_t)R * R);
  SPB_ALLOC(ar, double, Mf, (size_t)2 * R * k + 2 * (size_t)k * k);
  double* MfU = Mf;
  double* MfV = MfU + (size_t)R * k;
  double* EtfU = MfV + (size_t)R * k;
  double* EtfV = EtfU + (size_t)k * k;
  GramTail t1{dflag + 1, R1, R1i, dflag, 16.0 * R * 2.220446049250313e-16};
  GramTail t2{nullptr, nullptr, nullptr, nullptr, 0.0};
  if constexpr (R <= 8) {
    SPB_CUDA(launch_pdl((gram_stream_kernel<R>), dim3(nb), dim3(kGsThreads), 0, s, n, Y, (const double*)nullptr, P1, t1));
    SPB_CUDA(launch_pdl((gram_stream_kernel<R>), dim3(nb), dim3(kGsThreads), 0, s, n, Y, (const double*)R1i, P2, t2));
  } else {
    SPB_CUDA(launch_pdl((gram_rows_kernel<R>), dim3(nb), dim3(kGrThreads), 0, s, n, Y, nullptr, rpc, P1, t1));
    SPB_CUDA(launch_pdl((gram_rows_kernel<R>), dim3(nb), dim3(kGrThreads), 0, s, n, Y, R1i, rpc, P2, t2));
  }
  count_launch(2);
  SPB_CHECK_LAUNCH();
  const size_t fc_smem = (sizeof(FcShared) + 15) / 16 * 16 + (size_t)4 * k * R * sizeof(double);
  static int attr_dev = -1;  // once per device: host overhead is on the critical path here
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    SPB_CUDA(cudaFuncSetAttribute(finish_core_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    // fr_smem below reaches ~118 KB at (R, k) = (16, 256): allow the opt-in maximum
    SPB_CUDA(cudaFuncSetAttribute(finish_rows_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_dev = dev;
  }
  SPB_CUDA(launch_pdl((finish_core_kernel<R>), dim3(1), dim3(kFcThreads), fc_smem, s, k, nb, P2, R1, R1i, Z, ldz, Y, R, S, MfU, EtfU, MfV, EtfV,
                                                       dflag, hflag));
  count_launch();
  SPB_CHECK_LAUNCH();
  const int bu = ceil_div(m, kFrRows), bv = ceil_div(n, kFrRows);
  const size_t fr_smem =
      ((size_t)2 * R * k + R * R + (size_t)2 * kFrRows * R + (size_t)kFrRows * (R + 1)) * sizeof(double);
  // persistent: as many CTAs as fit walk the tiles (occupancy depends on k
  // through fr_smem: cached per k)
  static int fr_occ_k[257] = {0};
  int& fr_occ = fr_occ_k[k];
  if (fr_occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fr_occ, finish_rows_kernel<R>, kFrThreads, fr_smem) !=
            cudaSuccess ||
        fr_occ < 1)
      fr_occ = 1;
    cudaGetLastError();
  }
  const int fr_grid = (int)std::min<int64_t>((int64_t)bu + bv, (int64_t)fr_occ * kNumSMs);
  SPB_CUDA(launch_pdl((finish_rows_kernel<R>), dim3(fr_grid), dim3(kFrThreads), fr_smem, s, k, m, n, bu, Z, ldz, Y,
                      (int64_t)R, (const double*)R1i, (const double*)MfU, (const double*)EtfU, (const double*)MfV,
                      (const double*)EtfV, U, V));
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

// Y (n x r, ld r) = A^T Z is in place; writes U (m x k), S (k), V (n x k).
// dflag: device int[2] = {flag, ticket}, zero on entry; the flag is OR-ed on
// a Cholesky breakdown / non-finite input, published to *hflag (mapped pinned
// host memory, may be null) by finish_core and left zero for the next call.
int finish_fused(int64_t m, int64_t n, const double* Z, int64_t ldz, const double* Y, int r, int k, double* U,
                 double* S, double* V, int* dflag, int* hflag, cudaStream_t s) {
  SPB_REQUIRE(finish_fused_ok(m, n, r, k), "finish_fused limits exceeded");
  switch (r) {
#define SPB_FF(RR) \
  case RR:         \
    return finish_fused_r<RR>(m, n, Z, ldz, Y, k, U, S, V, dflag, hflag, s);
    SPB_FF(1) SPB_FF(2) SPB_FF(3) SPB_FF(4) SPB_FF(5) SPB_FF(6) SPB_FF(7) SPB_FF(8)
    SPB_FF(9) SPB_FF(10) SPB_FF(11) SPB_FF(12) SPB_FF(13) SPB_FF(14) SPB_FF(15) SPB_FF(16)
#undef SPB_FF
  }
  set_error("finish_fused: unsupported rank");
  return SP_ECONFIG;
}

}  // namespace spb
