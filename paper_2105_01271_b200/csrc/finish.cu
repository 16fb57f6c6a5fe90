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
//   tall_gram partials(Y) -> chol_small (shifted: R1, R1^{-1})
//   -> mul_gram (partial Gram of Q1 = Y R1^{-1}, Q1 never stored)
//   -> finish_core (1 CTA: Cholesky of Q1^T Q1 -> R2, R = R2 R1, Jacobi SVD
//      of R^T, the top k rows of both factors and both Householder
//      completions, concurrently in two thread groups)
//   -> finish_rows (one streaming pass writing U and V).
// No host synchronisation: the diagonal shift of the first Gram
// (16 r eps tr(G)) makes its Cholesky unconditionally defined, and the second
// pass restores O(eps) orthogonality for kappa(Y) up to ~1e7 (the caller
// routes kappa >= 1e6 to Householder TSQR).  A non-positive or non-finite
// pivot (non-finite A) raises a device flag the host reads lazily
// (sp_deferred_status) and S is poisoned with NaN.
#include "common.cuh"
#include "hh_complete.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

int chol_small_launch(int c, int nb, const double* P, double* R, double* Rinv, int* flag, double shift_rel,
                      cudaStream_t s);
int mul_gram_tiles(int64_t rows);
int mul_gram_launch(int64_t rows, int c, const double* X, int64_t ldx, const double* Ri, double* Q, int64_t ldq,
                    double* partial, int* nb_out, cudaStream_t s);

constexpr int kFcThreads = 512;
constexpr int kFcMaxR = 16;
constexpr double kFcJacTol = 1e-15;  // jacobi.cu kJacTol
constexpr int kFcMaxSweeps = 40;

struct FcShared {
  HcShared hc[2];                 // U / V completions
  double G[kFcMaxR][kFcMaxR + 1];  // Q1^T Q1 -> R2
  double R2i[kFcMaxR][kFcMaxR + 1];
  double R[kFcMaxR][kFcMaxR + 1];  // R = R2 R1
  double Us[kFcMaxR][kFcMaxR + 1];
  double Vs[kFcMaxR][kFcMaxR + 1];
  double Bv[kFcMaxR][kFcMaxR + 1];  // R2^{-1} Vs
  double R1i[kFcMaxR][kFcMaxR + 1];
  double red[kFcThreads];
  double sig[32];
  signed char ptab[31][32];
  int act[32], pos[32];
  int na, bad;
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
__device__ void fc_jacobi_warp(int r, double (&x)[RPW], double (&v)[RPW], FcShared& sh, int c) {
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
      const double hyp = (ad < 1e150 && ah < 1e150 && (ad > 1e-150 || ah > 1e-150)) ? sqrt(fma(d, d, h * h))
                                                                                  : hypot(d, h);
      const double t = copysign(1.0, d) * h / (ad + hyp);
      const double cs = rsqrt(fma(t, t, 1.0));
      const double sn = cs * t;
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

// S (k): sigma desc, zero padded; MfU / MfV (r x k), EtfU / EtfV (k x k):
// U = Z MfU + [EtfU; 0],  V = (Y R1^{-1}) MfV + [EtfV; 0].
// ws: scratch of 2 (k r + r (k-r) + k (k-r)) doubles.
template <int RPW>
__global__ void __launch_bounds__(kFcThreads)
finish_core_kernel(int r, int k, int nb2, const double* __restrict__ P2, const double* __restrict__ R1,
                   const double* __restrict__ R1i, const double* __restrict__ Z, int64_t ldz,
                   const double* __restrict__ Y, int64_t ldy, double* __restrict__ S, double* __restrict__ ws,
                   double* __restrict__ MfU, double* __restrict__ EtfU, double* __restrict__ MfV,
                   double* __restrict__ EtfV, int* flag) {
  extern __shared__ __align__(16) unsigned char fc_smem[];
  FcShared& sh = *reinterpret_cast<FcShared*>(fc_smem);
  const int tid = threadIdx.x, nout = r * r;
  if (tid == 0) sh.bad = 0;
  for (int e = tid; e < nout; e += kFcThreads) sh.R1i[e / r][e % r] = R1i[e];
  // (a) fixed-order reduction of the nb2 partial Grams of Q1
  {
    const int gs = kFcThreads / nout;  // >= 2 for r <= 16
    const int o = tid / gs, g = tid % gs;
    double a = 0.0;
    if (o < nout)
      for (int b = g; b < nb2; b += gs) a += P2[(int64_t)b * nout + o];
    sh.red[tid] = a;
    __syncthreads();
    if (g == 0 && o < nout) {
      double t = sh.red[tid];
      for (int q = 1; q < gs; ++q) t += sh.red[tid + q];
      sh.G[o / r][o % r] = t;
    }
    __syncthreads();
  }
  // (b) warp 0: Cholesky Q1^T Q1 = R2^T R2, R2^{-1}, R = R2 R1, Jacobi of R^T
  if (tid < 32) {
    const int lane = tid;
    bool bad = false;
    for (int j = 0; j < r; ++j) {
      const double d = sh.G[j][j];
      if (!(d > 0.0)) {
        bad = true;
        break;
      }
      const double dinv = 1.0 / d;
      const int w2 = r - j - 1;
      for (int e = lane; e < w2 * w2; e += 32) {
        const int i = j + 1 + e / w2, l = j + 1 + e % w2;
        if (l >= i) sh.G[i][l] = fma(-sh.G[j][i] * dinv, sh.G[j][l], sh.G[i][l]);
      }
      __syncwarp();
    }
    if (bad) {
      if (lane == 0) sh.bad = 1;
    } else {
      if (lane < r) sh.sig[lane] = sqrt(sh.G[lane][lane]);
      __syncwarp();
      for (int e = lane; e < nout; e += 32) {
        const int i = e / r, l = e % r;
        sh.G[i][l] = (l > i) ? sh.G[i][l] / sh.sig[i] : (l == i ? sh.sig[i] : 0.0);
      }
      __syncwarp();
      if (lane < r) {  // column l of R2^{-1} by back substitution
        const int l = lane;
        for (int i = r - 1; i >= 0; --i) {
          double acc = (i == l) ? 1.0 : 0.0;
          for (int q = i + 1; q <= l; ++q) acc = fma(-sh.G[i][q], sh.R2i[q][l], acc);
          sh.R2i[i][l] = (i <= l) ? acc / sh.G[i][i] : 0.0;
        }
      }
      for (int e = lane; e < nout; e += 32) {
        const int i = e / r, l = e % r;
        double acc = 0.0;
        for (int q = i; q <= l; ++q) acc = fma(sh.G[i][q], R1[q * r + l], acc);
        sh.R[i][l] = (l >= i) ? acc : 0.0;
      }
      __syncwarp();
      // M = R^T: lane c holds column c of M = row c of R
      double x[RPW], v[RPW];
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        x[i] = (i < r && lane < r) ? sh.R[lane][i] : 0.0;
        v[i] = (i == lane) ? 1.0 : 0.0;
      }
      fc_jacobi_warp<RPW>(r, x, v, sh, lane);
      double a1 = 0.0;
#pragma unroll
      for (int i = 0; i < RPW; ++i) a1 = fma(x[i], x[i], a1);
      const double sc = sqrt(a1);
      __syncwarp();
      sh.sig[lane] = lane < r ? sc : -1.0;
      __syncwarp();
      int rank = 0;
      for (int d = 0; d < 32; ++d) {
        const double sd = sh.sig[d];
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
  if (sh.bad) {
    if (tid == 0) atomicOr(flag, 1);
    for (int j = tid; j < k; j += kFcThreads) S[j] = __longlong_as_double(0x7ff8000000000000ll);
    return;  // uniform
  }
  // (c) Bv = R2^{-1} Vs; top k rows: XU = Z[0:k] Us, XV = (Y[0:k] R1^{-1}) Bv
  for (int e = tid; e < nout; e += kFcThreads) {
    const int i = e / r, l = e % r;
    double acc = 0.0;
    for (int q = i; q < r; ++q) acc = fma(sh.R2i[i][q], sh.Vs[q][l], acc);
    sh.Bv[i][l] = acc;
  }
  __syncthreads();
  const int kr = k - r;
  double* XU = ws;
  double* XV = XU + (size_t)k * r;
  double* KpU = XV + (size_t)k * r;
  double* KpV = KpU + (size_t)r * kr;
  double* EtU = KpV + (size_t)r * kr;
  double* EtV = EtU + (size_t)k * kr;
  for (int e = tid; e < k * r; e += kFcThreads) {
    const int i = e / r, l = e % r;
    double au = 0.0, av = 0.0;
    for (int p = 0; p < r; ++p) {
      au = fma(Z[(int64_t)i * ldz + p], sh.Us[p][l], au);
      // q1[i][p] in mul_gram's order (sum over the input columns from 0)
      double q1 = 0.0;
      for (int t = 0; t < r; ++t) q1 = fma(Y[(int64_t)i * ldy + t], sh.R1i[t][p], q1);
      av = fma(q1, sh.Bv[p][l], av);
    }
    XU[e] = au;
    XV[e] = av;
  }
  __syncthreads();
  // (d) both completions at once: threads [0, 256) -> U, [256, 512) -> V
  const int grp = tid >> 8;
  __shared__ double BuS[kFcMaxR * kFcMaxR], BvS[kFcMaxR * kFcMaxR];
  for (int e = tid; e < nout; e += kFcThreads) {
    BuS[e] = sh.Us[e / r][e % r];
    BvS[e] = sh.Bv[e / r][e % r];
  }
  __syncthreads();
  hh_complete_dev(r, k, grp ? XV : XU, r, grp ? KpV : KpU, grp ? EtV : EtU, kr, grp ? BvS : BuS, r,
                  grp ? MfV : MfU, grp ? EtfV : EtfU, sh.hc[grp], tid & 255, 256);
}

// One streaming pass: rows [0, m) of U (blocks [0, bu)) and [0, n) of V.
constexpr int kFrRows = 128;

__global__ void __launch_bounds__(kFrRows)
finish_rows_kernel(int r, int k, int64_t m, int64_t n, int bu, const double* __restrict__ Z, int64_t ldz,
                   const double* __restrict__ Y, int64_t ldy, const double* __restrict__ R1i,
                   const double* __restrict__ MfU, const double* __restrict__ EtfU, const double* __restrict__ MfV,
                   const double* __restrict__ EtfV, double* __restrict__ U, int64_t ldu, double* __restrict__ V,
                   int64_t ldv) {
  extern __shared__ __align__(16) double fr_smem[];
  double* mf = fr_smem;                    // r x k
  double* ri = mf + r * k;                 // r x r
  double* st = ri + kFcMaxR * kFcMaxR;     // kFrRows x 33 staging
  const bool isv = blockIdx.x >= bu;
  const int64_t rows = isv ? n : m;
  const int64_t base = (int64_t)(isv ? blockIdx.x - bu : blockIdx.x) * kFrRows;
  const double* X = isv ? Y : Z;
  const int64_t ldx = isv ? ldy : ldz;
  const double* Mf = isv ? MfV : MfU;
  const double* Et = isv ? EtfV : EtfU;
  double* O = isv ? V : U;
  const int64_t ldo = isv ? ldv : ldu;
  const int t = threadIdx.x;
  for (int e = t; e < r * k; e += kFrRows) cp_async_f64(&mf[e], Mf + e, true);
  if (isv)
    for (int e = t; e < r * r; e += kFrRows) cp_async_f64(&ri[e], R1i + e, true);
  const int nr = (int)imin64(kFrRows, rows - base);
  double x[kFcMaxR];
  const int64_t row = base + t;
#pragma unroll
  for (int i = 0; i < kFcMaxR; ++i) x[i] = (t < nr && i < r) ? X[row * ldx + i] : 0.0;
  cp_async_wait_all();
  __syncthreads();
  if (isv) {  // q1 = y R1^{-1}, mul_gram's summation order
    double q[kFcMaxR];
#pragma unroll
    for (int j = 0; j < kFcMaxR; ++j) q[j] = 0.0;
#pragma unroll
    for (int i = 0; i < kFcMaxR; ++i)
      if (i < r) {
#pragma unroll
        for (int j = 0; j < kFcMaxR; ++j)
          if (j < r) q[j] = fma(x[i], ri[i * r + j], q[j]);
      }
#pragma unroll
    for (int j = 0; j < kFcMaxR; ++j) x[j] = q[j];
  }
  const bool top = t < nr && row < k;
  for (int c0 = 0; c0 < k; c0 += 32) {
    const int cw = k - c0 < 32 ? k - c0 : 32;
    for (int cc = 0; cc < cw; ++cc) {
      double o = 0.0;
#pragma unroll
      for (int p = 0; p < kFcMaxR; ++p)
        if (p < r) o = fma(x[p], mf[p * k + c0 + cc], o);
      if (top) o += Et[row * k + c0 + cc];
      st[t * 33 + cc] = o;
    }
    __syncthreads();
    for (int e = t; e < nr * cw; e += kFrRows) {
      const int rl = e / cw, cl = e % cw;
      O[(base + rl) * ldo + c0 + cl] = st[rl * 33 + cl];
    }
    __syncthreads();
  }
}

bool finish_fused_ok(int64_t m, int64_t n, int r, int k) {
  return r >= 1 && r <= kFcMaxR && k >= r && k <= kHcMaxK && r * k <= 64 * 64 && m >= k && n >= k &&
         n >= 256;
}

// Y (n x r, ld r) = A^T Z is in place; writes U (m x k), S (k), V (n x k).
// dflag: device int, OR-ed on a Cholesky breakdown / non-finite input.
int finish_fused(int64_t m, int64_t n, const double* Z, int64_t ldz, const double* Y, int r, int k, double* U,
                 double* S, double* V, int* dflag, cudaStream_t s) {
  SPB_REQUIRE(finish_fused_ok(m, n, r, k), "finish_fused limits exceeded");
  Arena ar(s);
  const int nb1max = (int)std::min<int64_t>(4 * kNumSMs, ceil_div(n, 128));
  const int tiles = mul_gram_tiles(n);
  const int nb2 = ceil_div(n, (int64_t)128 * tiles);
  const int kr = k - r;
  SPB_ALLOC(ar, double, P1, (size_t)nb1max * r * r);
  SPB_ALLOC(ar, double, P2, (size_t)nb2 * r * r);
  SPB_ALLOC(ar, double, R1, (size_t)r * r);
  SPB_ALLOC(ar, double, R1i, (size_t)r * r);
  SPB_ALLOC(ar, double, Mf, (size_t)2 * r * k + 2 * (size_t)k * k);
  SPB_ALLOC(ar, double, ws, (size_t)2 * ((size_t)k * r + (size_t)r * kr + (size_t)k * kr));
  double* MfU = Mf;
  double* MfV = MfU + (size_t)r * k;
  double* EtfU = MfV + (size_t)r * k;
  double* EtfV = EtfU + (size_t)k * k;
  int nb1 = 0;
  SPB_TRY(tall_gram_partials(n, r, Y, r, r, Y, r, P1, nb1max, &nb1, s));
  SPB_TRY(chol_small_launch(r, nb1, P1, R1, R1i, dflag, 16.0 * r * 2.220446049250313e-16, s));
  int nb2o = 0;
  SPB_TRY(mul_gram_launch(n, r, Y, r, R1i, nullptr, r, P2, &nb2o, s));
  const size_t fc_smem = sizeof(FcShared);
  if (r <= 8) {
    SPB_CUDA(cudaFuncSetAttribute(finish_core_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fc_smem));
    finish_core_kernel<8><<<1, kFcThreads, fc_smem, s>>>(r, k, nb2o, P2, R1, R1i, Z, ldz, Y, r, S, ws, MfU, EtfU,
                                                         MfV, EtfV, dflag);
  } else {
    SPB_CUDA(cudaFuncSetAttribute(finish_core_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fc_smem));
    finish_core_kernel<16><<<1, kFcThreads, fc_smem, s>>>(r, k, nb2o, P2, R1, R1i, Z, ldz, Y, r, S, ws, MfU, EtfU,
                                                          MfV, EtfV, dflag);
  }
  count_launch();
  SPB_CHECK_LAUNCH();
  const int bu = ceil_div(m, kFrRows), bv = ceil_div(n, kFrRows);
  const size_t fr_smem = ((size_t)r * k + kFcMaxR * kFcMaxR + (size_t)kFrRows * 33) * sizeof(double);
  SPB_CUDA(cudaFuncSetAttribute(finish_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fr_smem));
  finish_rows_kernel<<<bu + bv, kFrRows, fr_smem, s>>>(r, k, m, n, bu, Z, ldz, Y, r, R1i, MfU, EtfU, MfV, EtfV,
                                                       U, k, V, k);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

}  // namespace spb
