// Nearly exactly rounded FP64 products on the DMMA pipe (Ozaki splitting).
//
// Why: the ID's enriched sketch E = C (C^T C) (src/power.py:282-285) feeds the
// greedy pivoted QR, whose pivots past the signal are decided by residual
// norms a few ulps apart.  The reference's own E (OpenBLAS, any kernel / thread
// count / association) is within ~1e-16 elementwise of the exact product and
// reproduces its 100 pivots at cfg3; an FP64 GEMM with another summation order
// lands ~1e-15 away and the pivots part at ~44 (measured: scripts/
// r2_pivot_probe.py; the K7 kernel itself matches the oracle's pivots on the
// same E exactly).  Computing E to ~2^-57 of its row x column scale makes the
// device pivots those of the exact product -- the reference's.
//
// Method (after Ozaki, Ogita, Oishi & Rump 2012): every row of op(A) and
// every column of B is cut into a head S0 / T0 of `bits` bits on a grid
// anchored at that row's / column's largest magnitude and a tail S1 = A - S0,
// T1 = B - T0 (|S1| < 2^-bits of the row scale).  With K 2^(2 bits) <= 2^53
// every partial sum of S0 T0 is an integer multiple of (unit_a x unit_b)
// below 2^53, so the level-0 product L0 = S0 T0 is EXACT in FP64 for any
// summation order (split-K, DMMA tile order, cross-rank allreduce).  The rest,
// L1 = S0 T1 + S1 B (one DMMA GEMM of depth 2K: [S0 | S1] [T1; B]), is about
// 2^-bits of the scale, so its FP64 rounding is ~2^-(53 + bits) of the scale.
// L0 + L1 summed in double-double: the product to ~2^-66 of sum |a_il||b_lj|
// at K = 5000, twice the FP64 work of a plain GEMM.
#include <cmath>

#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

__device__ __forceinline__ int exp_of(double mx) {
  int e = 0;
  frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1)  ->  mx < 2^e
  return mx > 0.0 ? e : 0;
}

// exponent of each row's (axis 1) / column's (axis 0) largest magnitude
__global__ void __launch_bounds__(256) row_exp_kernel(int64_t rows, int64_t cols, const double* __restrict__ X,
                                                      int64_t ldx, int* __restrict__ e) {
  __shared__ double red[8];
  const int64_t i = blockIdx.x;
  if (i >= rows) return;
  double mx = 0.0;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) mx = fmax(mx, fabs(X[i * ldx + j]));
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
    e[i] = mx > 0.0 ? exp_of(mx) : -100000;  // a zero row must not lift an allreduce-max
  }
}

// columns: 32 per block (threadIdx.x), rows strided over threadIdx.y and
// blockIdx.y; exp_of is monotone in the magnitude, so the per-column max
// exponent is an atomicMax of the partial ones (e preset below any exponent)
__global__ void col_exp_kernel(int64_t rows, int64_t cols, const double* __restrict__ X, int64_t ldx,
                               int* __restrict__ e) {
  __shared__ int part[8][32];
  const int64_t c = (int64_t)blockIdx.x * 32 + threadIdx.x;
  double mx = 0.0;
  if (c < cols)
    for (int64_t r = (int64_t)blockIdx.y * blockDim.y + threadIdx.y; r < rows; r += (int64_t)gridDim.y * blockDim.y)
      mx = fmax(mx, fabs(X[r * ldx + c]));
  part[threadIdx.y][threadIdx.x] = mx > 0.0 ? exp_of(mx) : -100000;
  __syncthreads();
  if (threadIdx.y == 0 && c < cols) {
    int m = part[0][threadIdx.x];
    for (int y = 1; y < (int)blockDim.y; ++y) m = max(m, part[y][threadIdx.x]);
    atomicMax(e + c, m);
  }
}

__device__ __forceinline__ void head_tail(double x, int e, int bits, double& h, double& t) {
  // a zero row / column (e below any real exponent) has head and tail 0
  const int sh = e - bits;
  h = (e < -90000) ? 0.0 : ldexp(trunc(ldexp(x, -sh)), sh);
  t = x - h;  // exact: h is x truncated to a coarser grid
}

// rows (exponent e[i]): out[i * ldo + j] = S0, out[i * ldo + cols + j] = S1
__global__ void __launch_bounds__(256) split_rows_kernel(int64_t rows, int64_t cols, const double* __restrict__ X,
                                                         int64_t ldx, const int* __restrict__ e, int bits,
                                                         double* __restrict__ out, int64_t ldo) {
  const int64_t i = blockIdx.x;
  if (i >= rows) return;
  const int ei = e[i];
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
    double h, t;
    head_tail(X[i * ldx + j], ei, bits, h, t);
    out[i * ldo + j] = h;
    out[i * ldo + cols + j] = t;
  }
}

// columns (exponent e[c]): head rows at out[r * ldo + c], tail rows at
// out[(rows + r) * ldo + c]; `copy` (may be null) receives X itself
__global__ void split_cols_kernel(int64_t rows, int64_t cols, const double* __restrict__ X, int64_t ldx,
                                  const int* __restrict__ e, int bits, double* __restrict__ out, int64_t ldo,
                                  double* __restrict__ copy, int64_t ldcp) {
  const int64_t c = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int64_t r = (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
  if (c >= cols || r >= rows) return;
  const double x = X[r * ldx + c];
  double h, t;
  head_tail(x, e[c], bits, h, t);
  out[r * ldo + c] = h;
  out[(rows + r) * ldo + c] = t;
  if (copy) copy[r * ldcp + c] = x;
}

// (hi, lo) = dd sum of the exact levels L[0..nl) (+ an inexact tail term t)
__global__ void dd_levels_kernel(int64_t M, int64_t N, const double* __restrict__ L, int nl, int64_t lstride,
                                 const double* __restrict__ tail, double* __restrict__ hi, double* __restrict__ lo,
                                 int64_t ldc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  double s = L[e], err = 0.0;
  for (int l = 1; l < nl; ++l) {
    const double x = L[(int64_t)l * lstride + e];
    const double t = s + x;
    const double bb = t - s;
    err += (s - (t - bb)) + (x - bb);
    s = t;
  }
  if (tail) err += tail[e];
  const double h = s + err;
  const int64_t o = (e / N) * ldc + (e % N);
  hi[o] = h;
  if (lo) lo[o] = err - (h - s);
}

// head width for an exact level-0 sum of depth K (K 2^(2 bits) <= 2^53); the
// product is always two levels (L0 exact, L1 the FP64 rest)
void ozaki_plan(int64_t K, int* bits_out, int* nsl_out) {
  const double need = std::ceil(std::log2((double)std::max<int64_t>(K, 1)));
  *bits_out = (int)std::floor((53.0 - need) / 2.0);
  *nsl_out = 2;
}

int row_exponents(int64_t rows, int64_t cols, const double* X, int64_t ldx, int* e, cudaStream_t s) {
  row_exp_kernel<<<(unsigned)rows, 256, 0, s>>>(rows, cols, X, ldx, e);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

int col_exponents(int64_t rows, int64_t cols, const double* X, int64_t ldx, int* e, cudaStream_t s) {
  SPB_CUDA(cudaMemsetAsync(e, 0x80, cols * sizeof(int), s));  // INT_MIN-ish: every exponent is larger
  dim3 g(ceil_div(cols, 32), std::min(ceil_div(rows, 64), 1024));
  col_exp_kernel<<<g, dim3(32, 8), 0, s>>>(rows, cols, X, ldx, e);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

// The levels of op(A) B on the slicing grids ea (per row of op(A)) and eb (per
// column of B): Lv[0] = S0 T0 (exact for any summation order: level sums of
// different ranks on the same grids -- allreduce-max of the exponents first --
// add up exactly when the total depth satisfies the plan), Lv[1] = the FP64 rest.
int gemm_exact_levels(int ta, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const int* ea,
                      const double* B, int64_t ldb, const int* eb, int bits, int nsl, double* Lv, cudaStream_t s,
                      bool symmetric) {
  SPB_REQUIRE(M >= 1 && N >= 1 && K >= 1 && nsl == 2, "gemm_exact_levels: bad extents");
  // symmetric: op(A) = B^T (the Gram T = C^T C): both operands get the same
  // slices (same vectors, same anchors), so the exact head level is exactly
  // symmetric and the rest level symmetric up to its own rounding -- only the
  // tiles on and above the diagonal are computed and mirrored
  symmetric = symmetric && ta == 1 && M == N;
  Arena ar(s);
  // A: [S0 | S1] along K
  const int64_t ka = 2 * K;
  SPB_ALLOC(ar, double, As, (size_t)M * ka);
  if (ta == 0) {
    split_rows_kernel<<<(unsigned)M, 256, 0, s>>>(M, K, A, lda, ea, bits, As, ka);  // M x 2K
  } else {
    dim3 g(ceil_div(M, 32), ceil_div(K, 8));
    split_cols_kernel<<<g, dim3(32, 8), 0, s>>>(K, M, A, lda, ea, bits, As, M, nullptr, 0);  // 2K x M
  }
  // B: [T0; T1; B] along K: level 0 takes rows [0, K), level 1 rows [K, 3K)
  SPB_ALLOC(ar, double, Bs, (size_t)3 * K * N);
  {
    dim3 g(ceil_div(N, 32), ceil_div(K, 8));
    split_cols_kernel<<<g, dim3(32, 8), 0, s>>>(K, N, B, ldb, eb, bits, Bs, N, Bs + 2 * K * N, N);
  }
  count_launch(2);
  SPB_CHECK_LAUNCH();
  double* L0 = Lv;
  double* L1 = Lv + (int64_t)M * N;
  if (ta == 0) {
    SPB_TRY(gemm(0, 0, M, N, K, 1.0, As, ka, Bs, N, 0.0, L0, N, s));
    SPB_TRY(gemm(0, 0, M, N, 2 * K, 1.0, As, ka, Bs + K * N, N, 0.0, L1, N, s));
  } else if (symmetric) {
    SPB_TRY(gemm_upper(1, 0, M, N, K, 1.0, As, M, Bs, N, 0.0, L0, N, s));
    SPB_TRY(gemm_upper(1, 0, M, N, 2 * K, 1.0, As, M, Bs + K * N, N, 0.0, L1, N, s));
    SPB_TRY(mirror_upper(M, L0, N, s));
    SPB_TRY(mirror_upper(M, L1, N, s));
  } else {
    SPB_TRY(gemm(1, 0, M, N, K, 1.0, As, M, Bs, N, 0.0, L0, N, s));
    SPB_TRY(gemm(1, 0, M, N, 2 * K, 1.0, As, M, Bs + K * N, N, 0.0, L1, N, s));
  }
  return SP_OK;
}

// (hi, lo) = double-double sum of the levels (+ an inexact tail term)
int dd_levels(int64_t M, int64_t N, const double* Lv, int nsl, const double* tail, double* hi, double* lo,
              int64_t ldc, cudaStream_t s) {
  dd_levels_kernel<<<ceil_div(M * N, 256), 256, 0, s>>>(M, N, Lv, nsl, M * N, tail, hi, lo, ldc);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

// C_hi (+ C_lo) = op(A) (B_hi + B_lo), nearly exactly rounded (error below
// 2^-(bits nsl) of sum_l |a_il| |b_lj|; with C_lo the result is a double-double).
// op(A) = A (ta = 0, M x K, lda) or A^T (ta = 1, A is K x M).  B is K x N (ldb),
// B_lo (same layout, may be null) the low part of a double-double B.
int gemm_exact(int ta, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B_hi,
               const double* B_lo, int64_t ldb, double* C_hi, double* C_lo, int64_t ldc, cudaStream_t s,
               bool symmetric) {
  SPB_REQUIRE(M >= 1 && N >= 1 && K >= 1, "gemm_exact needs non-empty operands");
  symmetric = symmetric && ta == 1 && M == N && B_lo == nullptr;
  int bits = 0, nsl = 0;
  ozaki_plan(K, &bits, &nsl);
  Arena ar(s);
  SPB_ALLOC(ar, int, ea, (size_t)M);
  SPB_ALLOC(ar, int, eb, (size_t)N);
  if (ta == 0)
    SPB_TRY(row_exponents(M, K, A, lda, ea, s));
  else
    SPB_TRY(col_exponents(K, M, A, lda, ea, s));
  SPB_TRY(col_exponents(K, N, B_hi, ldb, eb, s));
  SPB_ALLOC(ar, double, Lv, (size_t)nsl * M * N);
  SPB_TRY(gemm_exact_levels(ta, M, N, K, A, lda, ea, B_hi, ldb, eb, bits, nsl, Lv, s, symmetric));
  double* tail = nullptr;
  if (B_lo) {
    tail = ar.alloc<double>((size_t)M * N);
    if (!tail) {
      set_error("gemm_exact workspace allocation failed");
      return SP_ECUDA;
    }
    SPB_TRY(gemm(ta, 0, M, N, K, 1.0, A, lda, B_lo, ldb, 0.0, tail, N, s));
  }
  return dd_levels(M, N, Lv, nsl, tail, C_hi, C_lo, ldc, s);
}

}  // namespace spb
