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

// per-row grid: X (rows x cols, ldx) -> slices stacked along the columns:
// out[i * ldo + k * cols + j] (ldo >= nsl * cols)
__global__ void __launch_bounds__(256) split_rows_kernel(int64_t rows, int64_t cols, const double* __restrict__ X,
                                                         int64_t ldx, int bits, int nsl, double* __restrict__ out,
                                                         int64_t ldo) {
  __shared__ double red[8];
  const int64_t i = blockIdx.x;
  if (i >= rows) return;
  const double* x = X + i * ldx;
  double mx = 0.0;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) mx = fmax(mx, fabs(x[j]));
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
  const int e = exp_of(mx);
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) ozaki_slices(x[j], e, bits, nsl, out + i * ldo + j, cols);
}

// per-column grid: X (rows x cols, ldx) -> slices stacked along the rows:
// stacked position p holds slice p (rev = 0) or slice nsl - 1 - p (rev = 1):
// out[(p * rows + r) * ldo + c]
__global__ void __launch_bounds__(256) split_cols_kernel(int64_t rows, int64_t cols, const double* __restrict__ X,
                                                         int64_t ldx, int bits, int nsl, int rev,
                                                         double* __restrict__ out, int64_t ldo) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  double mx = 0.0;
  for (int64_t r = 0; r < rows; ++r) mx = fmax(mx, fabs(X[r * ldx + c]));
  const int e = exp_of(mx);
  double sl[8];
  for (int64_t r = 0; r < rows; ++r) {
    ozaki_slices(X[r * ldx + c], e, bits, nsl, sl, 1);
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
static void ozaki_plan(int64_t K, int& bits, int& nsl) {
  for (nsl = 3; nsl <= 6; ++nsl) {
    const double need = std::log2((double)nsl * (double)K);
    bits = (int)std::floor((53.0 - std::ceil(need)) / 2.0);
    if (bits * nsl >= 56) return;
  }
  nsl = 6;
}

// C_hi (+ C_lo) = op(A) (B_hi + B_lo), nearly exactly rounded (error below
// 2^-(bits nsl) of sum_l |a_il| |b_lj|; with C_lo the result is a double-double).
// op(A) = A (ta = 0, M x K, lda) or A^T (ta = 1, A is K x M).  B is K x N (ldb),
// B_lo (same layout, may be null) the low part of a double-double B.
int gemm_exact(int ta, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B_hi,
               const double* B_lo, int64_t ldb, double* C_hi, double* C_lo, int64_t ldc, cudaStream_t s) {
  SPB_REQUIRE(M >= 1 && N >= 1 && K >= 1, "gemm_exact needs non-empty operands");
  int bits = 0, nsl = 0;
  ozaki_plan(K, bits, nsl);
  Arena ar(s);
  // A slices: S_0..S_{nsl-1} concatenated along K
  const int64_t ka = (int64_t)nsl * K;
  SPB_ALLOC(ar, double, As, (size_t)M * ka);
  if (ta == 0) {
    split_rows_kernel<<<(unsigned)M, 256, 0, s>>>(M, K, A, lda, bits, nsl, As, ka);  // M x (nsl K)
  } else {
    split_cols_kernel<<<ceil_div(M, 256), 256, 0, s>>>(K, M, A, lda, bits, nsl, 0, As, M);  // (nsl K) x M
  }
  count_launch();
  SPB_CHECK_LAUNCH();
  // B slices stacked along K as [T_{nsl-1}; ...; T_1; T_0]: the level-L
  // operand is its last (L + 1) K rows, T_L ... T_0, pairing with A's
  // S_0 ... S_L (i + j = L)
  SPB_ALLOC(ar, double, Bs, (size_t)nsl * K * N);
  split_cols_kernel<<<ceil_div(N, 256), 256, 0, s>>>(K, N, B_hi, ldb, bits, nsl, 1, Bs, N);
  count_launch();
  SPB_CHECK_LAUNCH();
  SPB_ALLOC(ar, double, Lv, (size_t)nsl * M * N);
  for (int L = 0; L < nsl; ++L) {
    const int64_t depth = (int64_t)(L + 1) * K;
    const double* bop = Bs + (int64_t)(nsl - 1 - L) * K * N;
    if (ta == 0)
      SPB_TRY(gemm(0, 0, M, N, depth, 1.0, As, ka, bop, N, 0.0, Lv + (int64_t)L * M * N, N, s));
    else
      SPB_TRY(gemm(1, 0, M, N, depth, 1.0, As, M, bop, N, 0.0, Lv + (int64_t)L * M * N, N, s));
  }
  double* tail = nullptr;
  if (B_lo) {
    tail = ar.alloc<double>((size_t)M * N);
    if (!tail) {
      set_error("gemm_exact workspace allocation failed");
      return SP_ECUDA;
    }
    SPB_TRY(gemm(ta, 0, M, N, K, 1.0, A, lda, B_lo, ldb, 0.0, tail, N, s));
  }
  dd_levels_kernel<<<ceil_div(M * N, 256), 256, 0, s>>>(M, N, Lv, nsl, M * N, tail, C_hi, C_lo, ldc);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

}  // namespace spb
