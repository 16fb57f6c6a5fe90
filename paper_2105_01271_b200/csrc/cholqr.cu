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

// ------------------------------------------------ fused path, c <= 32 ----
// Five launches for CholeskyQR2 of a tall block with c <= 32 columns:
//   tall_gram partials(X) -> chol_small -> mul_gram (Q1 = X R1^{-1} and the
//   partial Gram of Q1 in the same pass) -> chol_small (R = R2 R1) -> tall_mul.
// Partials are summed in a fixed order: bitwise reproducible.
constexpr int kCsThreads = 1024;

// G = sum_b P[b] (nb slabs of c x c), Cholesky G = R^T R, Rinv = R^{-1};
// when R1 != nullptr also Rout = R R1 (upper triangular product).
__global__ void __launch_bounds__(kCsThreads)
chol_small_kernel(int c, int nb, const double* __restrict__ P, double* __restrict__ R, double* __restrict__ Rinv,
                  const double* __restrict__ R1, double* __restrict__ Rout, int64_t ldro, int* flag,
                  double shift_rel = 0.0) {
  __shared__ double G[32][33];
  __shared__ double Ri[32][33];
  __shared__ double part[8][32 * 32 / 8 + 1];
  const int tid = threadIdx.x, nout = c * c;
  SPB_TDECL;
  SPB_TMARK(0);
  // fixed-order reduction: thread (o, g) sums slabs g, g + G, ... of output o
  const int gsplit = kCsThreads / nout >= 32 ? 32 : (kCsThreads / nout >= 1 ? kCsThreads / nout : 1);
  for (int o0 = 0; o0 < nout; o0 += kCsThreads / gsplit) {
    const int o = o0 + tid / gsplit, g = tid % gsplit;
    double a = 0.0;
    if (o < nout && tid / gsplit < kCsThreads / gsplit) {
#pragma unroll 4
      for (int b = g; b < nb; b += gsplit) a += P[(int64_t)b * nout + o];
    }
    __shared__ double tmp[kCsThreads];
    tmp[tid] = a;
    __syncthreads();
    if (g == 0 && o < nout && tid / gsplit < kCsThreads / gsplit) {
      double t = tmp[tid];
      for (int q = 1; q < gsplit; ++q) t += tmp[tid + q];
      G[o / c][o % c] = t;
    }
    __syncthreads();
  }
  // the factorisation of the c x c core: warp 0 alone, warp-synchronous
  // (no block barriers on the critical path; the other warps are done)
  if (tid >= 32) return;
  const int lane = tid;
  SPB_TMARK(1);
  if (shift_rel > 0.0) {
    // shifted CholeskyQR: G + s I with s = shift_rel tr(G) (lane order sum,
    // identical in every lane) keeps the factorisation defined
    double tr = 0.0;
    for (int i = 0; i < c; ++i) tr += G[i][i];
    __syncwarp();
    if (lane < c) G[lane][lane] += shift_rel * tr;
    __syncwarp();
  }
  bool bad = false;
  for (int j = 0; j < c; ++j) {
    const double d = G[j][j];
    if (!(d > 0.0)) {  // uniform: every lane reads the same d
      bad = true;
      break;
    }
    const double dinv = 1.0 / d;
    const int w2 = c - j - 1;
    for (int e = lane; e < w2 * w2; e += 32) {
      const int i = j + 1 + e / w2, l = j + 1 + e % w2;
      if (l >= i) G[i][l] = fma(-G[j][i] * dinv, G[j][l], G[i][l]);
    }
    __syncwarp();
  }
  if (bad) {
    if (lane == 0) atomicOr(flag, 1);
    return;
  }
  __shared__ double dsq[32];
  if (lane < c) dsq[lane] = sqrt(G[lane][lane]);
  __syncwarp();
  for (int e = lane; e < nout; e += 32) {
    const int i = e / c, l = e % c;
    G[i][l] = (l > i) ? G[i][l] / dsq[i] : (l == i ? dsq[i] : 0.0);
  }
  __syncwarp();
  // R^{-1}: column l solved by lane l (back substitution, c <= 32)
  if (lane < c) {
    const int l = lane;
    for (int i = c - 1; i >= 0; --i) {
      double acc = (i == l) ? 1.0 : 0.0;
      for (int q = i + 1; q <= l; ++q) acc = fma(-G[i][q], Ri[q][l], acc);
      Ri[i][l] = (i <= l) ? acc / G[i][i] : 0.0;
    }
  }
  __syncwarp();
  for (int e = lane; e < nout; e += 32) {
    const int i = e / c, l = e % c;
    R[e] = G[i][l];
    Rinv[e] = Ri[i][l];
    if (Rout) {
      double acc = 0.0;
      for (int q = i; q <= l; ++q) acc = fma(G[i][q], R1[q * c + l], acc);
      Rout[(int64_t)i * ldro + l] = (l >= i) ? acc : 0.0;
    }
  }
  SPB_TMARK(2);
  if (lane == 0) SPB_TPRINT("chol_small reduce/factor", 3);
}

// Q1 rows = X rows R^{-1} (c x c) and partial[blk] = Q1_blk^T Q1_blk; one
// thread per row (c <= 32), rows staged through shared memory.
constexpr int kMgRows = 128;
// row tiles per CTA: at least 2, and enough that the partial count stays <= 2048
__host__ __device__ inline int mg_tiles(int64_t rows) {
  const int64_t t = (rows + (int64_t)128 * 2048 - 1) / ((int64_t)128 * 2048);
  return (int)(t < 2 ? 2 : t);
}

__global__ void __launch_bounds__(kMgRows)
mul_gram_kernel(int64_t rows, int c, const double* __restrict__ X, int64_t ldx, const double* __restrict__ Ri,
                double* __restrict__ Q, int64_t ldq, double* __restrict__ partial, int kMgTiles) {
  __shared__ double ms[32][32];
  __shared__ double ts[kMgRows][33];
  const int t = threadIdx.x;
  for (int e = t; e < c * c; e += kMgRows) cp_async_f64(&ms[e / c][e % c], Ri + e, true);
  // thread t accumulates Gram outputs t, t + 128, ... over the CTA's tiles
  double gacc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) gacc[u] = 0.0;
  for (int tile = 0; tile < kMgTiles; ++tile) {
    const int64_t base = ((int64_t)blockIdx.x * kMgTiles + tile) * kMgRows;
    if (base >= rows) break;  // uniform
    const int nr = (int)imin64(kMgRows, rows - base);
    if (t < nr) {  // thread per row: no division in the staging loop
      const double* src = X + (base + t) * ldx;
      for (int cc = 0; cc < c; ++cc) cp_async_f64(&ts[t][cc], src + cc, true);
    }
    cp_async_wait_all();
    __syncthreads();
    double acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0;
    if (t < nr) {
      for (int i = 0; i < c; ++i) {
        const double xi = ts[t][i];
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < c) acc[j] = fma(xi, ms[i][j], acc[j]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < c) ts[t][j] = t < nr ? acc[j] : 0.0;
    __syncthreads();
    if (Q != nullptr && t < nr) {
      double* dst = Q + (base + t) * ldq;
      for (int cc = 0; cc < c; ++cc) dst[cc] = ts[t][cc];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int o = t + u * kMgRows;
      if (o < c * c) {
        const int a = o / c, b = o % c;
        double s0 = 0.0, s1 = 0.0;
        int rr = 0;
        for (; rr + 1 < nr; rr += 2) {
          s0 = fma(ts[rr][a], ts[rr][b], s0);
          s1 = fma(ts[rr + 1][a], ts[rr + 1][b], s1);
        }
        if (rr < nr) s0 = fma(ts[rr][a], ts[rr][b], s0);
        gacc[u] += s0 + s1;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int o = t + u * kMgRows;
    if (o < c * c) partial[(int64_t)blockIdx.x * c * c + o] = gacc[u];
  }
}

// launch wrappers for the fused finish stage (finish.cu)
int chol_small_launch(int c, int nb, const double* P, double* R, double* Rinv, int* flag, double shift_rel,
                      cudaStream_t s) {
  chol_small_kernel<<<1, kCsThreads, 0, s>>>(c, nb, P, R, Rinv, nullptr, nullptr, 0, flag, shift_rel);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

int mul_gram_tiles(int64_t rows) { return mg_tiles(rows); }

// partial Grams of Q1 = X Ri (Q1 written to Q unless Q == nullptr); nb slabs
int mul_gram_launch(int64_t rows, int c, const double* X, int64_t ldx, const double* Ri, double* Q, int64_t ldq,
                    double* partial, int* nb_out, cudaStream_t s) {
  const int tiles = mg_tiles(rows);
  const int nb = ceil_div(rows, (int64_t)kMgRows * tiles);
  *nb_out = nb;
  mul_gram_kernel<<<nb, kMgRows, 0, s>>>(rows, c, X, ldx, Ri, Q, ldq, partial, tiles);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

static int cholqr2_small(int64_t rows, int c, const double* X, int64_t ldx, double* Q, int64_t ldq, double* R,
                         int64_t ldr, int* dflag, cudaStream_t s) {
  Arena ar(s);
  const int nb1 = (int)std::min<int64_t>(4 * kNumSMs, ceil_div(rows, 128));
  const int kMgTiles = mg_tiles(rows);
  const int nb2 = ceil_div(rows, (int64_t)kMgRows * kMgTiles);
  SPB_ALLOC(ar, double, P1, (size_t)nb1 * c * c);
  SPB_ALLOC(ar, double, P2, (size_t)nb2 * c * c);
  SPB_ALLOC(ar, double, R1, (size_t)c * c);
  SPB_ALLOC(ar, double, R1i, (size_t)c * c);
  SPB_ALLOC(ar, double, R2, (size_t)c * c);
  SPB_ALLOC(ar, double, R2i, (size_t)c * c);
  SPB_ALLOC(ar, double, Q1, (size_t)rows * c);
  int nb = 0;
  SPB_TRY(tall_gram_partials(rows, c, X, ldx, c, X, ldx, P1, nb1, &nb, s));
  chol_small_kernel<<<1, kCsThreads, 0, s>>>(c, nb, P1, R1, R1i, nullptr, nullptr, 0, dflag);
  count_launch();
  SPB_CHECK_LAUNCH();
  mul_gram_kernel<<<nb2, kMgRows, 0, s>>>(rows, c, X, ldx, R1i, Q1, c, P2, kMgTiles);
  count_launch();
  SPB_CHECK_LAUNCH();
  chol_small_kernel<<<1, kCsThreads, 0, s>>>(c, nb2, P2, R2, R2i, R1, R, ldr, dflag);
  count_launch();
  SPB_CHECK_LAUNCH();
  return tall_mul(rows, c, Q1, c, c, R2i, c, 1.0, 0.0, Q, ldq, s);
}

// CholeskyQR2.  Returns SP_OK with *breakdown = true when a Cholesky failed
// (Q, R are then garbage and the caller must fall back).  Synchronises once.
// Asynchronous CholeskyQR2: breakdown is OR-ed into the device flag *dflag
// (caller zeroes it and reads it later); no host synchronisation.
int cholqr2_async(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
                  double* R, int64_t ldr, int* dflag, cudaStream_t s) {
  SPB_REQUIRE(cols >= 1 && cols <= 112 && rows >= cols, "cholqr2 needs rows >= cols, cols <= 112");
  const int c = (int)cols;
  if (c <= 32 && rows >= 256) return cholqr2_small(rows, c, X, ldx, Q, ldq, R, ldr, dflag, s);
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
  SPB_TRY(read_small(&h, flag, sizeof(int), s));
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
