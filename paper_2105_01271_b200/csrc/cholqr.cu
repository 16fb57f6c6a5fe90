// CholeskyQR2 for WELL-CONDITIONED tall-skinny blocks (kappa < ~1e6):
// the orthonormal completions of the returned factors and the QR of the
// single-read output Y = A^T U_r when the kept spectrum spans < 1e6.
// Each pass: Gram on the DMMA GEMM (split-K), Cholesky + explicit R^{-1} of
// the c x c core in one CTA, Q = X R^{-1} on the DMMA GEMM.  Two passes give
// orthogonality O(eps) for kappa(X) < eps^{-1/2}.  Breakdown (non-positive
// pivot) is reported so callers can fall back to Householder TSQR.
#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

// G (c x c, ld c) -> R upper with R^T R = G and Rinv = R^{-1}; flag=1 on breakdown
__global__ void chol_inv_kernel(int c, const double* __restrict__ Gin, double* __restrict__ R,
                                double* __restrict__ Rinv, int* flag) {
  extern __shared__ double sm[];
  double* G = sm;          // c x c working copy (upper part used)
  double* Ri = sm + c * c;  // c x c inverse
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < c * c; e += nt) {
    G[e] = Gin[e];
    Ri[e] = 0.0;
  }
  __syncthreads();
  __shared__ int bad;
  if (tid == 0) bad = 0;
  __syncthreads();
  // Unscaled right-looking elimination: step j updates rows i > j with
  // G[i][l] -= G[j][i] G[j][l] / G[j][j] (row j itself is final after step
  // j-1), one __syncthreads per step; rows are scaled by 1/sqrt(G[j][j]) at
  // the end.
  for (int j = 0; j < c; ++j) {
    const double d = G[j * c + j];
    if (!(d > 0.0)) {
      if (tid == 0) bad = 1;
      break;  // uniform: every thread reads the same d
    }
    const double dinv = 1.0 / d;
    // 32 x 32 thread grid, element (i, l) owned by thread (i % 32, l % 32)
    const int ty = tid >> 5, tx = tid & 31;
    for (int i = j + 1 + ((ty - (j + 1)) % 32 + 32) % 32; i < c; i += 32) {
      const double gji = G[j * c + i] * dinv;
      for (int l = tx; l < c; l += 32)
        if (l >= i) G[i * c + l] = fma(-gji, G[j * c + l], G[i * c + l]);
    }
    __syncthreads();
  }
  __syncthreads();
  if (bad) {
    if (tid == 0) *flag = 1;
    return;
  }
  __shared__ double dsq[112];
  for (int i = tid; i < c; i += nt) dsq[i] = sqrt(G[i * c + i]);
  __syncthreads();
  for (int e = tid; e < c * c; e += nt) {
    const int i = e / c, l = e % c;
    if (l >= i) G[e] = (l == i) ? dsq[i] : G[e] / dsq[i];
  }
  __syncthreads();
  // R (upper) out; R^{-1} by recursive doubling: with the diagonal blocks of
  // size s inverted, each pair [A B; 0 C] gets its off-diagonal block
  // -A^{-1} B C^{-1}; log2(c) levels of block products, two syncs each.
  // T = B C^{-1} is parked transposed in the (unused) lower triangle of Ri.
  for (int e = tid; e < c * c; e += nt) {
    const int i = e / c, l = e % c;
    R[e] = (l >= i) ? G[e] : 0.0;
    if (i == l) Ri[e] = 1.0 / G[e];
  }
  __syncthreads();
  for (int sz = 1; sz < c; sz <<= 1) {
    // phase 1: T[b0+i][b0+sz+j] = sum_{l<=j} R[b0+i][b0+sz+l] Ri[b0+sz+l][b0+sz+j]
    const int pairs = (c + 2 * sz - 1) / (2 * sz);
    for (int e = tid; e < pairs * sz * sz; e += nt) {
      const int pb = e / (sz * sz), rem = e % (sz * sz), i = rem / sz, j = rem % sz;
      const int b0 = pb * 2 * sz, row = b0 + i, col = b0 + sz + j;
      if (col >= c) continue;
      double acc = 0.0;
      for (int l = 0; l <= j; ++l) acc = fma(G[row * c + b0 + sz + l], Ri[(b0 + sz + l) * c + col], acc);
      Ri[col * c + row] = acc;  // transposed park (lower triangle)
    }
    __syncthreads();
    // phase 2: Ri[b0+i][b0+sz+j] = -sum_{l>=i} Ri[b0+i][b0+l] T[b0+l][b0+sz+j]
    for (int e = tid; e < pairs * sz * sz; e += nt) {
      const int pb = e / (sz * sz), rem = e % (sz * sz), i = rem / sz, j = rem % sz;
      const int b0 = pb * 2 * sz, row = b0 + i, col = b0 + sz + j;
      if (col >= c) continue;
      double acc = 0.0;
      for (int l = i; l < sz; ++l) acc = fma(Ri[row * c + b0 + l], Ri[col * c + b0 + l], acc);
      Ri[row * c + col] = -acc;
    }
    __syncthreads();
  }
  for (int e = tid; e < c * c; e += nt) {
    const int i = e / c, l = e % c;
    Rinv[e] = (l >= i) ? Ri[e] : 0.0;
  }
}

// One CholeskyQR pass: Q = X R^{-1}, R from chol(X^T X).
static int cholqr_pass(int64_t rows, int c, const double* X, int64_t ldx, double* Q, int64_t ldq,
                       double* R, int* flag, Arena& ar, cudaStream_t s) {
  double* G = ar.alloc<double>((size_t)c * c);
  double* Ri = ar.alloc<double>((size_t)c * c);
  if (!G || !Ri) {
    set_error("cholqr workspace allocation failed");
    return SP_ECUDA;
  }
  SPB_TRY(gemm(1, 0, c, c, rows, 1.0, X, ldx, X, ldx, 0.0, G, c, s));
  const size_t smem = (size_t)2 * c * c * sizeof(double);
  SPB_CUDA(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  chol_inv_kernel<<<1, 1024, smem, s>>>(c, G, R, Ri, flag);
  count_launch();
  SPB_CHECK_LAUNCH();
  SPB_TRY(gemm(0, 0, rows, c, c, 1.0, X, ldx, Ri, c, 0.0, Q, ldq, s));
  return SP_OK;
}

// CholeskyQR2.  Returns SP_OK with *breakdown = true when a Cholesky failed
// (Q, R are then garbage and the caller must fall back).  Synchronises once.
// Asynchronous CholeskyQR2: breakdown is OR-ed into the device flag *dflag
// (caller zeroes it and reads it later); no host synchronisation.
int cholqr2_async(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
                  double* R, int64_t ldr, int* dflag, cudaStream_t s) {
  SPB_REQUIRE(cols >= 1 && cols <= 112 && rows >= cols, "cholqr2 needs rows >= cols, cols <= 112");
  const int c = (int)cols;
  Arena ar(s);
  SPB_ALLOC(ar, double, Q1, (size_t)rows * c);
  SPB_ALLOC(ar, double, R1, (size_t)c * c);
  SPB_ALLOC(ar, double, R2, (size_t)c * c);
  SPB_TRY(cholqr_pass(rows, c, X, ldx, Q1, c, R1, dflag, ar, s));
  SPB_TRY(cholqr_pass(rows, c, Q1, c, Q, ldq, R2, dflag, ar, s));
  SPB_TRY(gemm(0, 0, c, c, c, 1.0, R2, c, R1, c, 0.0, R, ldr, s));
  return SP_OK;
}

int cholqr2(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
            double* R, int64_t ldr, bool* breakdown, cudaStream_t s) {
  Arena ar(s);
  SPB_ALLOC(ar, int, flag, 1);
  SPB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  SPB_TRY(cholqr2_async(rows, cols, X, ldx, Q, ldq, R, ldr, flag, s));
  int h = 0;
  SPB_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  SPB_CUDA(cudaStreamSynchronize(s));
  *breakdown = (h != 0);
  return SP_OK;
}

// QR of a tall block: CholeskyQR2 when the caller certifies kappa < ~1e6 and
// the width fits, Householder TSQR otherwise or on breakdown.
int qr_tall(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq, double* R,
            int64_t ldr, bool well_conditioned, cudaStream_t s) {
  if (well_conditioned && cols <= 112 && rows >= cols) {
    bool bd = false;
    SPB_TRY(cholqr2(rows, cols, X, ldx, Q, ldq, R, ldr, &bd, s));
    if (!bd) return SP_OK;
  }
  return tsqr(rows, cols, X, ldx, Q, ldq, R, ldr, s);
}

}  // namespace spb
