// Small dense helpers of the path: sign convention, pseudo-inverse
// reciprocals, triangular solve, transposes, random blocks, thin QR / SVD
// drivers, streamed residual norm.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

// ------------------------------------------------------------ launches ----
#define SPB_LAUNCHED() \
  do {                 \
    count_launch();    \
    SPB_CHECK_LAUNCH(); \
  } while (0)

// --------------------------------------------------------- elementwise ----
__global__ void transpose_kernel(int64_t rows, int64_t cols, const double* __restrict__ X, int64_t ldx,
                                 double* __restrict__ Y, int64_t ldy) {
  __shared__ double tile[32][33];
  const int64_t tiles_x = (cols + 31) / 32;  // linear tile index: no 65535 limit on either side
  const int64_t bx = ((int64_t)blockIdx.x % tiles_x) * 32, by = ((int64_t)blockIdx.x / tiles_x) * 32;
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int64_t r = by + k, c = bx + threadIdx.x;
    tile[k][threadIdx.x] = (r < rows && c < cols) ? X[r * ldx + c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int64_t r = bx + k, c = by + threadIdx.x;  // Y is cols x rows
    if (r < cols && c < rows) Y[r * ldy + c] = tile[threadIdx.x][k];
  }
}

int transpose(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Y, int64_t ldy,
              cudaStream_t s) {
  if (rows == 0 || cols == 0) return SP_OK;
  dim3 g((unsigned)((int64_t)ceil_div(cols, 32) * ceil_div(rows, 32))), b(32, 8);
  transpose_kernel<<<g, b, 0, s>>>(rows, cols, X, ldx, Y, ldy);
  SPB_LAUNCHED();
  return SP_OK;
}

__global__ void copy2d_kernel(int64_t rows, int64_t cols, const double* __restrict__ X, int64_t ldx,
                              double* __restrict__ Y, int64_t ldy) {
  SPB_PDL_ENTRY();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  Y[(e / cols) * ldy + (e % cols)] = X[(e / cols) * ldx + (e % cols)];
}

int copy2d(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Y, int64_t ldy,
           cudaStream_t s) {
  if (rows == 0 || cols == 0) return SP_OK;
  SPB_CUDA(launch_pdl((copy2d_kernel), dim3(ceil_div(rows * cols, 256)), dim3(256), 0, s, rows, cols, X, ldx, Y, ldy));
  SPB_LAUNCHED();
  return SP_OK;
}

// X = rows [row_offset, row_offset + rows) of the seed's (.. x cols) uniform
// block: a rank holding a slab of a globally indexed random test block
// generates exactly its rows.
__global__ void fill_uniform_kernel(int64_t rows, int64_t cols, double* X, int64_t ldx, uint64_t seed,
                                    int64_t row_offset) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  X[(e / cols) * ldx + (e % cols)] = hash_uniform(seed, (uint64_t)(e + row_offset * cols));
}

int fill_uniform(int64_t rows, int64_t cols, double* X, int64_t ldx, uint64_t seed, cudaStream_t s,
                 int64_t row_offset) {
  if (rows == 0 || cols == 0) return SP_OK;
  fill_uniform_kernel<<<ceil_div(rows * cols, 256), 256, 0, s>>>(rows, cols, X, ldx, seed, row_offset);
  SPB_LAUNCHED();
  return SP_OK;
}

// max |X_ij| (non-negative doubles order like their int64 bit patterns, so an
// integer atomicMax is exact and order independent)
__global__ void max_abs_kernel(int64_t rows, int64_t cols, const double* X, int64_t ldx,
                               unsigned long long* out) {
  double mx = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols;
       e += (int64_t)gridDim.x * blockDim.x)
    mx = fmax(mx, fabs(X[(e / cols) * ldx + (e % cols)]));
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(mx));
}

int max_abs(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* out, cudaStream_t s) {
  SPB_CUDA(cudaMemsetAsync(out, 0, sizeof(double), s));
  if (rows == 0 || cols == 0) return SP_OK;
  const int grid = std::min(ceil_div(rows * cols, 256), 4 * kNumSMs);
  max_abs_kernel<<<grid, 256, 0, s>>>(rows, cols, X, ldx, reinterpret_cast<unsigned long long*>(out));
  SPB_LAUNCHED();
  return SP_OK;
}

__global__ void fill_uniform_scaled_kernel(int64_t rows, int64_t cols, double* X, int64_t ldx, uint64_t seed,
                                           const double* scale, double factor) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const double sc = *scale > 0.0 ? *scale * factor : 1.0;
  X[(e / cols) * ldx + (e % cols)] = hash_uniform(seed, (uint64_t)e) * sc;
}

int fill_uniform_scaled(int64_t rows, int64_t cols, double* X, int64_t ldx, uint64_t seed, const double* scale,
                        double factor, cudaStream_t s) {
  if (rows == 0 || cols == 0) return SP_OK;
  fill_uniform_scaled_kernel<<<ceil_div(rows * cols, 256), 256, 0, s>>>(rows, cols, X, ldx, seed, scale, factor);
  SPB_LAUNCHED();
  return SP_OK;
}

__global__ void scale_cols_kernel(int64_t rows, int64_t cols, double* X, int64_t ldx, const double* d) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  X[(e / cols) * ldx + (e % cols)] *= d[e % cols];
}

int scale_cols(int64_t rows, int64_t cols, double* X, int64_t ldx, const double* d, cudaStream_t s) {
  if (rows == 0 || cols == 0) return SP_OK;
  scale_cols_kernel<<<ceil_div(rows * cols, 256), 256, 0, s>>>(rows, cols, X, ldx, d);
  SPB_LAUNCHED();
  return SP_OK;
}

__global__ void div_cols_kernel(int64_t rows, int64_t cols, double* X, int64_t ldx, const double* d) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  X[(e / cols) * ldx + (e % cols)] /= d[e % cols];
}

// X[:, j] /= d[j] (the vt /= s_k of direct_svd, src/svd.py:113) or *= d[j]
int scale_columns(int64_t rows, int64_t cols, double* X, int64_t ldx, const double* d, bool divide, cudaStream_t s) {
  if (rows == 0 || cols == 0) return SP_OK;
  if (!divide) return scale_cols(rows, cols, X, ldx, d, s);
  div_cols_kernel<<<ceil_div(rows * cols, 256), 256, 0, s>>>(rows, cols, X, ldx, d);
  SPB_LAUNCHED();
  return SP_OK;
}

// out[i, :] = X[idx[i], :] (k x cols, widened to f64): the fine skeleton rows
// of the two-pass IDs (src/rowid.py:82-95)
template <typename T>
__global__ void gather_rows_any(const T* __restrict__ X, int64_t ldx, int64_t cols, const int64_t* __restrict__ idx,
                                int64_t k, double* __restrict__ out, int64_t ldo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * cols) return;
  const int64_t i = e / cols, j = e % cols;
  out[i * ldo + j] = (double)X[idx[i] * ldx + j];
}

int gather_rows(const void* X, int dtype, int64_t ldx, int64_t cols, const int64_t* idx, int64_t k, double* out,
                int64_t ldo, cudaStream_t s) {
  if (k == 0 || cols == 0) return SP_OK;
  if (dtype == SP_F64)
    gather_rows_any<double><<<ceil_div(k * cols, 256), 256, 0, s>>>((const double*)X, ldx, cols, idx, k, out, ldo);
  else if (dtype == SP_F32)
    gather_rows_any<float><<<ceil_div(k * cols, 256), 256, 0, s>>>((const float*)X, ldx, cols, idx, k, out, ldo);
  else {
    set_error("unknown dtype tag");
    return SP_ECONFIG;
  }
  SPB_LAUNCHED();
  return SP_OK;
}

__global__ void all_finite_kernel(int64_t rows, int64_t cols, const double* X, int64_t ldx, int* bad) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  if (!isfinite(X[(e / cols) * ldx + (e % cols)])) atomicOr(bad, 1);
}

// OR 1 into *dflag when X holds a NaN/Inf (no synchronisation)
int check_finite_async(int64_t rows, int64_t cols, const double* X, int64_t ldx, int* dflag, cudaStream_t s) {
  if (rows == 0 || cols == 0) return SP_OK;
  all_finite_kernel<<<ceil_div(rows * cols, 256), 256, 0, s>>>(rows, cols, X, ldx, dflag);
  SPB_LAUNCHED();
  return SP_OK;
}

// Synchronises; returns SP_ENUMERICAL with `what` in the message on NaN/Inf.
int check_finite(int64_t rows, int64_t cols, const double* X, int64_t ldx, const char* what,
                 cudaStream_t s) {
  if (rows == 0 || cols == 0) return SP_OK;
  Arena ar(s);
  SPB_ALLOC(ar, int, bad, 1);
  SPB_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  all_finite_kernel<<<ceil_div(rows * cols, 256), 256, 0, s>>>(rows, cols, X, ldx, bad);
  SPB_LAUNCHED();
  int h = 0;
  SPB_TRY(read_small(&h, bad, sizeof(int), s));
  if (h) {
    set_error(std::string(what));
    return SP_ENUMERICAL;
  }
  return SP_OK;
}

// ------------------------------------------------------ sign convention ----
// src/kernels.py:52-71: flip column j so its first entry with |x| > 1e-12 *
// max|x| is >= 0; companions flip the same column ("col") or row ("row").
__global__ void sign_fix_kernel(int64_t rows, const double* __restrict__ basis_in, double* basis,
                                int64_t ldb, double* comp, int64_t ldc, int64_t comp_len, int comp_row) {
  __shared__ double red[32];
  __shared__ long long first_s[32];
  const int j = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double peak = 0.0;
  for (int64_t i = tid; i < rows; i += blockDim.x) peak = fmax(peak, fabs(basis[i * ldb + j]));
  peak = warp_max(peak);
  if (lane == 0) red[warp] = peak;
  __syncthreads();
  peak = 0.0;
  for (int w = 0; w < nw; ++w) peak = fmax(peak, red[w]);
  if (peak == 0.0) return;  // uniform
  long long first = rows;
  for (int64_t i = tid; i < rows; i += blockDim.x)
    if (fabs(basis[i * ldb + j]) > 1e-12 * peak) {
      first = i;
      break;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
  if (lane == 0) first_s[warp] = first;
  __syncthreads();
  first = rows;
  for (int w = 0; w < nw; ++w) first = min(first, first_s[w]);
  if (first >= rows) return;  // cannot happen when peak > 0
  const bool flip = basis[first * ldb + j] < 0.0;
  __syncthreads();
  if (!flip) return;
  for (int64_t i = tid; i < rows; i += blockDim.x) basis[i * ldb + j] = -basis[i * ldb + j];
  if (comp) {
    if (comp_row)
      for (int64_t c = tid; c < comp_len; c += blockDim.x) comp[(int64_t)j * ldc + c] = -comp[(int64_t)j * ldc + c];
    else
      for (int64_t i = tid; i < comp_len; i += blockDim.x) comp[i * ldc + j] = -comp[i * ldc + j];
  }
}

int sign_fix(int64_t rows, int64_t cols, double* basis, int64_t ldb, double* comp, int64_t ldc,
             int64_t comp_len, bool comp_row, cudaStream_t s) {
  if (cols == 0 || rows == 0) return SP_OK;
  sign_fix_kernel<<<(int)cols, 256, 0, s>>>(rows, basis, basis, ldb, comp, ldc, comp_len, comp_row ? 1 : 0);
  SPB_LAUNCHED();
  return SP_OK;
}

// ---------------------------------------------------------- pinv_apply ----
// src/kernels.py:158-168 (the non-increasing precondition is checked by the
// host mirror, as in the reference).
__global__ void pinv_kernel(const double* s, int64_t n, double tol, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double s0 = s[0];
  out[i] = (s0 != 0.0 && s[i] > tol * s0) ? 1.0 / s[i] : 0.0;
}

int pinv_apply(const double* s, int64_t n, double tol, double* out, cudaStream_t st) {
  if (n == 0) return SP_OK;
  pinv_kernel<<<ceil_div(n, 256), 256, 0, st>>>(s, n, tol, out);
  SPB_LAUNCHED();
  return SP_OK;
}

// ------------------------------------------------------- triangular solve ----
// X = R^{-1} B, R upper triangular k x k; one thread per right-hand side
// column, back substitution in the order of LAPACK's dtrsv.
__global__ void trsm_upper_kernel(int64_t k, const double* __restrict__ R, int64_t ldr, int64_t ncols,
                                  const double* __restrict__ B, int64_t ldb, double* X, int64_t ldx) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  for (int64_t i = k - 1; i >= 0; --i) {
    double acc = B[i * ldb + c];
    for (int64_t j = i + 1; j < k; ++j) acc = fma(-R[i * ldr + j], X[j * ldx + c], acc);
    X[i * ldx + c] = acc / R[i * ldr + i];
  }
}

int trsm_upper(int64_t k, const double* R, int64_t ldr, int64_t ncols, const double* B, int64_t ldb,
               double* X, int64_t ldx, cudaStream_t s) {
  if (k == 0 || ncols == 0) return SP_OK;
  trsm_upper_kernel<<<ceil_div(ncols, 128), 128, 0, s>>>(k, R, ldr, ncols, B, ldb, X, ldx);
  SPB_LAUNCHED();
  return SP_OK;
}

// -------------------------------------------------------- thin QR / SVD ----
// Sketch-sized cores (p <= 256) keep the round-1 path; wider inputs (the
// drop-in thin_qr / thin_svd on whole sketches: 2000 x 4096 ... 10000 x 16384)
// take the size-general one below.
constexpr int64_t kSmallCore = 256;

// out (N x k, ld ldo): columns [0, r) orthonormal; columns [r, k) receive an
// orthonormal completion (Householder reconstruction when small, else the
// Q factor of [out_r | uniform] by the panel TSQR).
int complete_basis(int64_t N, int r, int k, double* out, int64_t ldo, uint64_t seed, cudaStream_t s) {
  if (r >= k) return SP_OK;
  if (householder_complete(N, r, k, out, ldo, s) == SP_OK) return SP_OK;
  Arena ar(s);
  SPB_ALLOC(ar, double, W, (size_t)N * k);
  SPB_ALLOC(ar, double, Qc, (size_t)N * k);
  SPB_ALLOC(ar, double, Rc, (size_t)k * k);
  if (r > 0) SPB_TRY(copy2d(N, r, out, ldo, W, k, s));
  SPB_TRY(fill_uniform(N, k - r, W + r, k, seed, s));
  SPB_TRY(tsqr(N, k, W, k, Qc, k, Rc, k, s));
  SPB_TRY(copy2d(N, k - r, Qc + r, k, out + r, ldo, s));
  return SP_OK;
}

// The one-sided Jacobi leaves the columns it never rotated (norm below
// 1e-15 ||M||_F, i.e. S_i ~ 0) unnormalised and not orthogonal to the rest:
// replace the left factor's columns past the last S_i > 1e-15 ||S||_2-sum by
// an orthonormal completion (the reference's gesdd returns a full orthonormal
// U for a rank-deficient input).  Synchronises (reads S).
int block_jacobi_svd(int64_t N, int64_t n, const double* M, int64_t ldm, bool trans, double* U, int64_t ldu,
                     double* S, double* V, int64_t ldv, cudaStream_t s);

__global__ void row_sumsq_kernel(int64_t rows, int64_t cols, const double* __restrict__ X, int64_t ldx,
                                 double* __restrict__ out) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  double a = 0.0;
  for (int64_t c = lane; c < cols; c += 32) a = fma(X[r * ldx + c], X[r * ldx + c], a);
  a = warp_sum(a);
  if (lane == 0) out[r] = a;
}

// Columns of M^T (rows of M, p x p) the one-sided Jacobi would rotate: squared
// norm above 1e-30 of the total (the negligibility rule of jacobi.cu).  Synchronises.
static int active_rows(int64_t p, const double* M, int64_t ldm, int64_t* count, cudaStream_t s) {
  Arena ar(s);
  SPB_ALLOC(ar, double, nr, (size_t)p);
  row_sumsq_kernel<<<ceil_div(p * 32, 256), 256, 0, s>>>(p, p, M, ldm, nr);
  SPB_LAUNCHED();
  std::vector<double> h((size_t)p);
  SPB_TRY(read_small(h.data(), nr, p * sizeof(double), s));
  double fro = 0.0;
  for (double x : h) fro += x;
  int64_t c = 0;
  for (double x : h) c += x > 1e-30 * fro ? 1 : 0;
  *count = c;
  return SP_OK;
}

// SVD of M^T for a p x p core M (the rows of M are the Jacobi columns):
// M^T = U S V^T.  More than kBlockJacobiMin active columns: the block Jacobi
// (bjacobi.cu, nb - 1 rounds per sweep); otherwise the scalar one-sided Jacobi
// (jacobi.cu), which skips the negligible columns and is faster for few.
constexpr int64_t kBlockJacobiMin = 512;
static int core_svd_rows(int64_t p, const double* M, int64_t ldm, double* U, int64_t ldu, double* S, double* V,
                         int64_t ldv, cudaStream_t s) {
  int64_t act = p;
  if (p > kBlockJacobiMin) SPB_TRY(active_rows(p, M, ldm, &act, s));
  if (act > kBlockJacobiMin) return block_jacobi_svd(p, p, M, ldm, /*trans=*/true, U, ldu, S, V, ldv, s);
  return jacobi_svd_tr(p, M, ldm, /*trans=*/true, U, ldu, S, V, ldv, s);
}

// out[:, c0:c1) = Q[:, c0:c1) with column j negated where R_jj < 0
__global__ void copy_signed_cols_kernel(int64_t rows, int64_t c0, int64_t c1, const double* __restrict__ Q,
                                        int64_t ldq, const double* __restrict__ R, int64_t ldr,
                                        double* __restrict__ out, int64_t ldo) {
  const int64_t w = c1 - c0;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * w) return;
  const int64_t i = e / w, j = c0 + e % w;
  const double q = Q[i * ldq + j];
  out[i * ldo + j] = R[j * ldr + j] < 0.0 ? -q : q;
}

static int complete_null_columns(int64_t p, const double* S, double* Ucols, int64_t ldu, cudaStream_t s,
                                 bool* all_zero = nullptr) {
  if (all_zero) *all_zero = false;
  std::vector<double> hs((size_t)p);
  SPB_TRY(read_small(hs.data(), S, p * sizeof(double), s));
  double fro2 = 0.0;
  for (double x : hs) fro2 += x * x;
  const double thr = 1e-15 * std::sqrt(fro2);
  int64_t r = 0;
  while (r < p && hs[r] > thr) ++r;
  if (r == 0) {  // the zero matrix: any orthonormal basis
    if (all_zero) *all_zero = true;
    SPB_CUDA(cudaMemset2DAsync(Ucols, ldu * sizeof(double), 0, p * sizeof(double), p, s));
    return fill_identity((int)p, Ucols, ldu, s);
  }
  // Graded spectra.  A normalised column w_j / S_j of the rotated core carries
  // the absolute rounding error ~eps S_1 of w_j, i.e. a relative error
  // ~eps S_1 / S_j: without a grading of the core itself (a Haar-mixed
  // spectrum down to 1e-13 S_1) the columns of the small S_j come out 1e-3
  // away from orthogonal to the rest (scripts/fuzz_dense.py seed 30873:
  // 300 x 256, U^T U - I = 9e-4), where LAPACK's U is orthonormal to eps.
  // Columns with S_j < 1e-6 S_1 (error above the 1e-10 contract) are
  // re-orthonormalised against the accurate leading ones and each other:
  // Householder QR of the first r columns, the Q columns taken with the sign
  // of R_jj.  The leading columns are left as they are (their R block is I to
  // rounding); the replaced ones move by their own error, which changes the
  // reconstruction by ~eps S_1.
  int64_t r0 = 0;
  while (r0 < r && hs[r0] >= 1e-6 * hs[0]) ++r0;
  if (r0 < r) {
    Arena ar(s);
    SPB_ALLOC(ar, double, Qc, (size_t)p * r);
    SPB_ALLOC(ar, double, Rc, (size_t)r * r);
    SPB_TRY(tsqr(p, r, Ucols, ldu, Qc, r, Rc, r, s));
    copy_signed_cols_kernel<<<ceil_div(p * (r - r0), 256), 256, 0, s>>>(p, r0, r, Qc, r, Rc, r, Ucols, ldu);
    SPB_LAUNCHED();
  }
  return complete_basis(p, (int)r, (int)p, Ucols, ldu, 0x5eedC0DEull, s);
}

// out (rows x p) = [I; 0]: the long factor of the zero matrix (its QR factor may
// repeat columns: an exactly zero panel of the multi-panel TSQR has no direction
// of its own)
static int fill_eye_tall(int64_t rows, int64_t p, double* out, int64_t ldo, cudaStream_t s) {
  SPB_CUDA(cudaMemset2DAsync(out, ldo * sizeof(double), 0, p * sizeof(double), rows, s));
  return fill_identity((int)p, out, ldo, s);
}

// src/kernels.py:74-84 thin_qr: Q rows x p, R p x cols, p = min(rows, cols)
int thin_qr(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
            double* R, int64_t ldr, cudaStream_t s) {
  SPB_REQUIRE(rows >= 1 && cols >= 1, "thin_qr needs a non-empty matrix");
  SPB_TRY(check_finite(rows, cols, X, ldx, "QR input contains non-finite entries", s));
  const int64_t p = std::min(rows, cols);
  if (rows >= cols) {
    SPB_TRY(tsqr(rows, cols, X, ldx, Q, ldq, R, ldr, s));
  } else {
    // X = [X1 X2] with X1 square: X1 = Q R1, R = [R1, Q^T X2]
    SPB_TRY(tsqr(rows, rows, X, ldx, Q, ldq, R, ldr, s));
    SPB_TRY(gemm(1, 0, rows, cols - rows, rows, 1.0, Q, ldq, X + rows, ldx, 0.0, R + rows, ldr, s));
  }
  SPB_TRY(sign_fix(rows, p, Q, ldq, R, ldr, cols, true, s));
  return SP_OK;
}

// src/kernels.py:87-94 thin_svd: U rows x p, S p, V cols x p
int thin_svd(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* U, int64_t ldu,
             double* S, double* V, int64_t ldv, cudaStream_t s) {
  SPB_REQUIRE(rows >= 1 && cols >= 1, "thin_svd needs a non-empty matrix");
  const int64_t p = std::min(rows, cols);
  SPB_TRY(check_finite(rows, cols, X, ldx, "SVD input contains non-finite entries", s));
  Arena ar(s);
  SPB_ALLOC(ar, double, Q, (size_t)std::max(rows, cols) * p);
  SPB_ALLOC(ar, double, R, (size_t)p * p);
  SPB_ALLOC(ar, double, Rt, (size_t)p * p);
  SPB_ALLOC(ar, double, Us, (size_t)p * p);
  SPB_ALLOC(ar, double, Vs, (size_t)p * p);
  if (rows >= cols && p > kSmallCore) {
    // X = Q R; one-sided Jacobi on the ROWS of R (the columns of R^T):
    // R^T = U' S V'^T  ->  X = (Q V') S U'^T, so U = Q V' (rotations, always
    // orthonormal) and V = U' (normalised rows, completed where S ~ 0).  The
    // rows of R beyond the numerical rank are rounding-sized and never enter
    // the Jacobi schedule, so a low-rank sketch costs rounds only for its rank.
    SPB_TRY(tsqr(rows, cols, X, ldx, Q, p, R, p, s));
    SPB_TRY(core_svd_rows(p, R, p, V, ldv, S, Us, p, s));
    bool zero = false;
    SPB_TRY(complete_null_columns(p, S, V, ldv, s, &zero));
    if (zero)
      SPB_TRY(fill_eye_tall(rows, p, U, ldu, s));
    else
      SPB_TRY(gemm(0, 0, rows, p, p, 1.0, Q, p, Us, p, 0.0, U, ldu, s));
  } else if (rows >= cols) {
    // X = Q R, R = Us S Vs^T  ->  U = Q Us, V = Vs
    SPB_TRY(tsqr(rows, cols, X, ldx, Q, p, R, p, s));
    SPB_TRY(jacobi_svd(p, R, p, Us, p, S, Vs, p, s));
    // Us holds the NORMALISED columns of the rotated R: where S ~ 0 they are
    // rounding noise (or zero), not an orthonormal completion as LAPACK's U is
    bool zero = false;
    SPB_TRY(complete_null_columns(p, S, Us, p, s, &zero));
    if (zero)
      SPB_TRY(fill_eye_tall(rows, p, U, ldu, s));
    else
      SPB_TRY(gemm(0, 0, rows, p, p, 1.0, Q, p, Us, p, 0.0, U, ldu, s));
    SPB_TRY(copy2d(p, p, Vs, p, V, ldv, s));
  } else {
    SPB_ALLOC(ar, double, Xt, (size_t)cols * rows);
    SPB_TRY(transpose(rows, cols, X, ldx, Xt, rows, s));
    return thin_svd_t(rows, cols, Xt, rows, U, ldu, S, V, ldv, s);
  }
  SPB_TRY(sign_fix(rows, p, U, ldu, V, ldv, cols, false, s));
  return SP_OK;
}

// thin_svd of X (rows x cols, rows <= cols) given Xt = X^T (cols x rows):
// the wide branch without the transpose -- the projected matrix of the
// two-pass SVDs arrives as (Q^T A)^T = A^T Q from the A pass.
// X^T = Q R  ->  X = R^T Q^T, R^T = Us S Vs^T  ->  U = Us, V = Q Vs
int thin_svd_t(int64_t rows, int64_t cols, const double* Xt, int64_t ldxt, double* U, int64_t ldu, double* S,
               double* V, int64_t ldv, cudaStream_t s) {
  SPB_REQUIRE(rows >= 1 && cols >= rows, "thin_svd_t needs 1 <= rows <= cols");
  SPB_TRY(check_finite(cols, rows, Xt, ldxt, "SVD input contains non-finite entries", s));
  const int64_t p = rows;
  Arena ar(s);
  SPB_ALLOC(ar, double, Q, (size_t)cols * p);
  SPB_ALLOC(ar, double, R, (size_t)p * p);
  SPB_ALLOC(ar, double, Rt, (size_t)p * p);
  SPB_ALLOC(ar, double, Vs, (size_t)p * p);
  SPB_TRY(tsqr(cols, rows, Xt, ldxt, Q, p, R, p, s));
  bool zero = false;
  if (p > kSmallCore) {
    // X^T = Q R -> X = R^T Q^T; SVD of R^T by Jacobi on the rows of R
    SPB_TRY(core_svd_rows(p, R, p, U, ldu, S, Vs, p, s));
    SPB_TRY(complete_null_columns(p, S, U, ldu, s, &zero));
  } else {
    SPB_TRY(transpose(p, p, R, p, Rt, p, s));
    SPB_TRY(jacobi_svd(p, Rt, p, U, ldu, S, Vs, p, s));
    SPB_TRY(complete_null_columns(p, S, U, ldu, s, &zero));  // normalised columns: noise where S ~ 0
  }
  if (zero)
    SPB_TRY(fill_eye_tall(cols, p, V, ldv, s));
  else
    SPB_TRY(gemm(0, 0, cols, p, p, 1.0, Q, p, Vs, p, 0.0, V, ldv, s));
  SPB_TRY(sign_fix(rows, p, U, ldu, V, ldv, cols, false, s));
  return SP_OK;
}

// ------------------------------------------------------ K8 residual norm ----
// err2 = sum_ij (A_ij - sum_c U_ic S_c V_jc)^2, ref2 = sum_ij A_ij^2.
// One thread per column j holds V[j, :] in shared memory (dynamic, k <= 256);
// rows are streamed with U S of the current row broadcast from shared memory.
// The verify pass of the CLI (src/cli.py:125-139) fused into one A read.
constexpr int kResThreads = 64;
constexpr int kResMaxK = 256;

template <typename TA>
__global__ void __launch_bounds__(kResThreads)
residual_kernel(const TA* __restrict__ A, int64_t m, int64_t n, int64_t lda, const double* __restrict__ U,
                int64_t ldu, const double* __restrict__ S, const double* __restrict__ V, int64_t ldv,
                int k, int64_t rows_per_cta, double* partial) {
  extern __shared__ double res_smem[];
  double* vs = res_smem;                           // [kResThreads][k + 1]
  double* us = res_smem + kResThreads * (k + 1);   // [k]
  __shared__ double red[2][kResThreads / 32];
  const int64_t j = (int64_t)blockIdx.x * kResThreads + threadIdx.x;
  for (int c = 0; c < k; ++c) vs[threadIdx.x * (k + 1) + c] = (j < n) ? V[j * ldv + c] : 0.0;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_cta, r1 = min(m, r0 + rows_per_cta);
  double e2 = 0.0, a2 = 0.0;
  for (int64_t i = r0; i < r1; ++i) {
    __syncthreads();
    for (int c = threadIdx.x; c < k; c += kResThreads) us[c] = U[i * ldu + c] * S[c];
    __syncthreads();
    if (j < n) {
      double rec = 0.0;
      const double* vr = vs + threadIdx.x * (k + 1);
      for (int c = 0; c < k; ++c) rec = fma(us[c], vr[c], rec);
      const double a = widen(A[i * lda + j]);
      const double d = a - rec;
      e2 = fma(d, d, e2);
      a2 = fma(a, a, a2);
    }
  }
  e2 = warp_sum(e2);
  a2 = warp_sum(a2);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = e2;
    red[1][threadIdx.x >> 5] = a2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double te = 0.0, ta = 0.0;
    for (int w = 0; w < kResThreads / 32; ++w) {
      te += red[0][w];
      ta += red[1][w];
    }
    const int64_t b = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
    partial[2 * b] = te;
    partial[2 * b + 1] = ta;
  }
}

int frob_residual(const void* A, int a_dtype, int64_t m, int64_t n, int64_t lda, const double* U,
                  int64_t ldu, const double* S, const double* V, int64_t ldv, int k, double* out2,
                  cudaStream_t s) {
  SPB_REQUIRE(k >= 0 && k <= kResMaxK, "frob_residual supports k <= 256");
  const int gx = ceil_div(n, kResThreads);
  int gy = std::max(1, std::min<int>(ceil_div(4 * kNumSMs, gx), (int)m));
  const int64_t rpc = ceil_div(m, gy);
  gy = ceil_div(m, rpc);
  Arena ar(s);
  SPB_ALLOC(ar, double, part, (size_t)2 * gx * gy);
  dim3 g(gx, gy);
  const size_t smem = ((size_t)kResThreads * (k + 1) + (size_t)std::max(k, 1)) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    SPB_CUDA(cudaFuncSetAttribute(residual_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    SPB_CUDA(cudaFuncSetAttribute(residual_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    attr = true;
  }
  if (a_dtype == SP_F64)
    residual_kernel<double><<<g, kResThreads, smem, s>>>((const double*)A, m, n, lda, U, ldu, S, V, ldv, k, rpc,
                                                         part);
  else
    residual_kernel<float><<<g, kResThreads, smem, s>>>((const float*)A, m, n, lda, U, ldu, S, V, ldv, k, rpc,
                                                        part);
  SPB_LAUNCHED();
  std::vector<double> h((size_t)2 * gx * gy);
  SPB_CUDA(cudaMemcpyAsync(h.data(), part, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  SPB_CUDA(cudaStreamSynchronize(s));
  double e = 0.0, a = 0.0;
  for (size_t b = 0; b < h.size() / 2; ++b) {
    e += h[2 * b];
    a += h[2 * b + 1];
  }
  out2[0] = e;
  out2[1] = a;
  return SP_OK;
}

}  // namespace spb
