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
// Method (Ozaki, Ogita, Oishi & Rump 2012): every row of op(A) and every
// column of B is cut into `nsl` slices of `bits` bits on a grid anchored at
// that row's / column's largest magnitude, so every slice product is an
// integer multiple of (unit_a x unit_b) below 2^(2 bits); with
// (L + 1) K 2^(2 bits) <= 2^53 the level-L sum  sum_{i+j=L} S_i^A S_j^B  (one
// DMMA GEMM of depth (L + 1) K, slices concatenated along K) is EXACT in FP64,
// whatever the summation order.  Levels 0..nsl-1 are summed in double-double;
// the dropped levels (i + j >= nsl) are below 2^-(bits nsl) of the scale.
#include <cmath>

#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

// slice k of x on the unit grid 2^(e - bits (k + 1)), e = exponent of the
// row / column max (max < 2^e); the last slice keeps the remainder
__device__ __forceinline__ void ozaki_slices(double x, int e, int bits, int nsl, double* out, int64_t stride) {
  double rem = x;
  for (int k = 0; k < nsl; ++k) {
    const int sh = e - bits * (k + 1);
    double sl = ldexp(trunc(ldexp(rem, -sh)), sh);
    if (k == nsl - 1) sl = rem;
    out[(int64_t)k * stride] = sl;
    rem -= sl;  // exact: sl is rem truncated to a coarser grid
  }
}

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
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
    mx = fmax(mx, red[0]);
    e[i] = exp_of(mx);
  }
}

__global__ void __launch_bounds__(256) col_exp_kernel(int64_t rows, int64_t cols, const double* __restrict__ X,
                                                      int64_t ldx, int* __restrict__ e) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  double mx = 0.0;
  for (int64_t r = 0; r < rows; ++r) mx = fmax(mx, fabs(X[r * ldx + c]));
  e[c] = exp_of(mx);
}

// per-row grid (exponent e[i]): slices of row i stacked along the columns,
// out[i * ldo + k * cols + j] (ldo >= nsl * cols)
__global__ void __launch_bounds__(256) split_rows_kernel(int64_t rows, int64_t cols, const double* __restrict__ X,
                                                         int64_t ldx, const int* __restrict__ e, int bits, int nsl,
                                                         double* __restrict__ out, int64_t ldo) {
  const int64_t i = blockIdx.x;
  if (i >= rows) return;
  const int ei = e[i];
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x)
    ozaki_slices(X[i * ldx + j], ei, bits, nsl, out + i * ldo + j, cols);
}

// per-column grid (exponent e[c]): slices stacked along the rows; stacked
// position p holds slice p (rev = 0) or slice nsl - 1 - p (rev = 1):
// out[(p * rows + r) * ldo + c]
__global__ void __launch_bounds__(256) split_cols_kernel(int64_t rows, int64_t cols, const double* __restrict__ X,
                                                         int64_t ldx, const int* __restrict__ e, int bits, int nsl,
                                                         int rev, double* __restrict__ out, int64_t ldo) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const int ec = e[c];
  double sl[8];
  for (int64_t r = 0; r < rows; ++r) {
    ozaki_slices(X[r * ldx + c], ec, bits, nsl, sl, 1);
    for (int p = 0; p < nsl; ++p) out[((int64_t)p * rows + r) * ldo + c] = sl[rev ? nsl - 1 - p : p];
  }
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

// slices / bits for an exact level sum of depth up to nsl * K
void ozaki_plan(int64_t K, int* bits_out, int* nsl_out) {
  int bits = 0, nsl = 3;
  for (; nsl <= 6; ++nsl) {
    const double need = std::log2((double)nsl * (double)K);
    bits = (int)std::floor((53.0 - std::ceil(need)) / 2.0);
    if (bits * nsl >= 56) break;
  }
  *bits_out = bits;
  *nsl_out = std::min(nsl, 6);
}

int row_exponents(int64_t rows, int64_t cols, const double* X, int64_t ldx, int* e, cudaStream_t s) {
  row_exp_kernel<<<(unsigned)rows, 256, 0, s>>>(rows, cols, X, ldx, e);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

int col_exponents(int64_t rows, int64_t cols, const double* X, int64_t ldx, int* e, cudaStream_t s) {
  col_exp_kernel<<<ceil_div(cols, 256), 256, 0, s>>>(rows, cols, X, ldx, e);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

// The exact levels Lv[L] (M x N each, L < nsl) of op(A) B on the slicing grids
// ea (per row of op(A)) and eb (per column of B): every level is an exact FP64
// value for ANY summation order, so level sums of different ranks (same grids:
// allreduce-max of the exponents first) add up exactly as long as the total
// depth K_total satisfies the plan for K_total.
int gemm_exact_levels(int ta, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const int* ea,
                      const double* B, int64_t ldb, const int* eb, int bits, int nsl, double* Lv, cudaStream_t s) {
  SPB_REQUIRE(M >= 1 && N >= 1 && K >= 1 && nsl >= 1 && nsl <= 6, "gemm_exact_levels: bad extents");
  Arena ar(s);
  // A slices: S_0..S_{nsl-1} concatenated along K
  const int64_t ka = (int64_t)nsl * K;
  SPB_ALLOC(ar, double, As, (size_t)M * ka);
  if (ta == 0)
    split_rows_kernel<<<(unsigned)M, 256, 0, s>>>(M, K, A, lda, ea, bits, nsl, As, ka);  // M x (nsl K)
  else
    split_cols_kernel<<<ceil_div(M, 256), 256, 0, s>>>(K, M, A, lda, ea, bits, nsl, 0, As, M);  // (nsl K) x M
  // B slices stacked along K as [T_{nsl-1}; ...; T_1; T_0]: the level-L
  // operand is its last (L + 1) K rows, T_L ... T_0, pairing with A's
  // S_0 ... S_L (i + j = L)
  SPB_ALLOC(ar, double, Bs, (size_t)nsl * K * N);
  split_cols_kernel<<<ceil_div(N, 256), 256, 0, s>>>(K, N, B, ldb, eb, bits, nsl, 1, Bs, N);
  count_launch(2);
  SPB_CHECK_LAUNCH();
  for (int L = 0; L < nsl; ++L) {
    const int64_t depth = (int64_t)(L + 1) * K;
    const double* bop = Bs + (int64_t)(nsl - 1 - L) * K * N;
    if (ta == 0)
      SPB_TRY(gemm(0, 0, M, N, depth, 1.0, As, ka, bop, N, 0.0, Lv + (int64_t)L * M * N, N, s));
    else
      SPB_TRY(gemm(1, 0, M, N, depth, 1.0, As, M, bop, N, 0.0, Lv + (int64_t)L * M * N, N, s));
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
               const double* B_lo, int64_t ldb, double* C_hi, double* C_lo, int64_t ldc, cudaStream_t s) {
  SPB_REQUIRE(M >= 1 && N >= 1 && K >= 1, "gemm_exact needs non-empty operands");
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
  SPB_TRY(gemm_exact_levels(ta, M, N, K, A, lda, ea, B_hi, ldb, eb, bits, nsl, Lv, s));
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
