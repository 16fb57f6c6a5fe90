// K4: Householder TSQR for tall-skinny matrices (<= 32 columns per panel).
//
// Replaces thin_qr / np.linalg.qr (src/kernels.py:74-84) on the path.  The
// sketch bases on this path are numerically rank deficient (SURVEY.md 7 "Hard
// parts"): CholeskyQR breaks down, so orthogonalisation is Householder
// based, which keeps the span of every direction to eps * ||X|| regardless of
// conditioning.
//
// Layout: a CTA factors a 256 x 32 chunk with LANE = COLUMN: warp w holds
// rows [32w, 32w+32) and lane c holds those 32 entries of column c in
// registers.  Loads / stores of a row are coalesced (lanes = consecutive
// columns), a column dot product is a private 32-term FMA chain plus an
// 8-way shared-memory reduction across warps, the reflector column is
// broadcast through shared memory -- two __syncthreads per Householder step
// and no predicated all-column sweeps.  Fixed reduction order, so results
// are bitwise reproducible.  The 32 x 32 R factors of the chunks are stacked
// and factored again until one chunk remains; Q is then formed top-down by
// applying each chunk's reflectors to its block of the parent Q.
#include "common.cuh"
#include "launch_count.cuh"

#include <vector>

namespace spb {

int gemm(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
         cudaStream_t s);

constexpr int kQB = 32;                 // panel width
constexpr int kQWarps = 8;
constexpr int kQThreads = kQWarps * 32;
constexpr int kQCH = kQWarps * 32;      // rows per chunk

// Row mapping: local row g = 8*i + w lives in warp w, register slot i, so
// the 32 diagonal rows are spread 4 per warp (slots 0..3): only those slots
// need j-dependent masks, every other slot is strictly below every diagonal.
__device__ __forceinline__ int qrow(int i, int w) { return i * kQWarps + w; }
constexpr int kQDiagSlots = kQB / kQWarps;  // 4

// Factor chunk blockIdx.x of X (rows x cols, cols <= 32).  Writes the
// reflectors (strictly below the chunk diagonal) to V (rows x 32), tau to
// tau[chunk*32 + j] and the chunk's upper-trapezoidal R into
// Rs[chunk*32 .. +32) x 32 (zero padded).
__global__ void __launch_bounds__(kQThreads)
tsqr_leaf_kernel(const double* __restrict__ X, int64_t rows, int cols, int64_t ldx, double* __restrict__ V,
                 double* __restrict__ tau, double* __restrict__ Rs) {
  __shared__ double colj[kQCH];
  __shared__ double part[kQWarps];
  __shared__ double red[kQWarps][kQB];
  __shared__ double rdiag[kQB];
  __shared__ double alpha_s;
  const int w = threadIdx.x >> 5, c = threadIdx.x & 31;
  const int64_t c0 = (int64_t)blockIdx.x * kQCH;
  const int nrow = (int)imin64(kQCH, rows - c0);
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int g = qrow(i, w);
    x[i] = (g < nrow && c < cols) ? X[(c0 + g) * ldx + c] : 0.0;
  }
  const int nref = nrow < kQB ? nrow : kQB;
  for (int j = 0; j < nref; ++j) {
    // (1) lane j publishes column j below the diagonal (zero on and above it)
    if (c == j) {
      double sq0 = 0.0, sq1 = 0.0;
#pragma unroll
      for (int i = 0; i < kQDiagSlots; ++i) {
        const int g = qrow(i, w);
        const double xi = (g > j) ? x[i] : 0.0;
        colj[g] = xi;
        sq0 = fma(xi, xi, sq0);
        if (g == j) alpha_s = x[i];
      }
#pragma unroll
      for (int i = kQDiagSlots; i < 32; i += 2) {
        colj[qrow(i, w)] = x[i];
        colj[qrow(i + 1, w)] = x[i + 1];
        sq0 = fma(x[i], x[i], sq0);
        sq1 = fma(x[i + 1], x[i + 1], sq1);
      }
      part[w] = sq0 + sq1;
    }
    __syncthreads();
    double sigma2 = 0.0;
#pragma unroll
    for (int q = 0; q < kQWarps; ++q) sigma2 += part[q];
    const double alpha = alpha_s;
    double beta = alpha, tj = 0.0, inv = 0.0;
    if (sigma2 > 0.0) {
      const double nrm = sqrt(fma(alpha, alpha, sigma2));
      beta = alpha >= 0.0 ? -nrm : nrm;
      tj = (beta - alpha) / beta;
      inv = 1.0 / (alpha - beta);
    }
    // (2) reflector entries of my rows (v_j = 1) and the dot with my column
    double v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = colj[qrow(i, w)] * inv;
#pragma unroll
    for (int i = 0; i < kQDiagSlots; ++i)
      if (qrow(i, w) == j) v[i] = 1.0;
    double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      p0 = fma(v[i], x[i], p0);
      p1 = fma(v[i + 1], x[i + 1], p1);
      p2 = fma(v[i + 2], x[i + 2], p2);
      p3 = fma(v[i + 3], x[i + 3], p3);
    }
    red[w][c] = (p0 + p1) + (p2 + p3);
    __syncthreads();
    double wc = 0.0;
#pragma unroll
    for (int q = 0; q < kQWarps; ++q) wc += red[q][c];
    wc *= tj;
    // (3) apply H_j to the trailing columns; lane j stores the reflector
    if (c > j) {
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = fma(-v[i], wc, x[i]);
    } else if (c == j) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int g = qrow(i, w);
        if (g < nrow) V[(c0 + g) * kQB + j] = (g > j) ? v[i] : 0.0;
      }
    }
    if (threadIdx.x == 0) {
      tau[(int64_t)blockIdx.x * kQB + j] = tj;
      rdiag[j] = beta;
    }
  }
  __syncthreads();
  // columns >= nref were never reflected: their reflector column is zero
  if (c >= nref) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int g = qrow(i, w);
      if (g < nrow) V[(c0 + g) * kQB + c] = 0.0;
    }
  }
  if (threadIdx.x < kQB && threadIdx.x >= nref) tau[(int64_t)blockIdx.x * kQB + threadIdx.x] = 0.0;
#pragma unroll
  for (int i = 0; i < kQDiagSlots; ++i) {
    const int g = qrow(i, w);  // g < 32
    double rv = 0.0;
    if (g < nrow && c >= g) rv = (c == g && g < nref) ? rdiag[g] : x[i];
    Rs[((int64_t)blockIdx.x * kQB + g) * kQB + c] = rv;
  }
}

// Out rows of chunk blockIdx.x = H_0 ... H_31 [Bin_chunk ; 0], where
// Bin_chunk = Bin[chunk*32 .. +32) (ld 32), or the identity when Bin == nullptr.
// The chunk's reflectors are staged once in shared memory (dynamic, 64 KB);
// one __syncthreads per reflector (reduction buffer double-buffered).
__global__ void __launch_bounds__(kQThreads)
tsqr_apply_kernel(const double* __restrict__ V, const double* __restrict__ tau, int64_t rows,
                  const double* __restrict__ Bin, double* __restrict__ Out, int64_t ldo, int out_cols) {
  extern __shared__ double vsm[];  // [kQCH][kQB]
  __shared__ double red[2][kQWarps][kQB];
  __shared__ double tau_s[kQB];
  const int w = threadIdx.x >> 5, c = threadIdx.x & 31;
  const int64_t c0 = (int64_t)blockIdx.x * kQCH;
  const int nrow = (int)imin64(kQCH, rows - c0);
  for (int e = threadIdx.x; e < kQCH * kQB; e += kQThreads) {
    const int g = e / kQB;
    vsm[e] = (g < nrow) ? V[(c0 + g) * kQB + (e % kQB)] : 0.0;
  }
  if (threadIdx.x < kQB) tau_s[threadIdx.x] = tau[(int64_t)blockIdx.x * kQB + threadIdx.x];
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int g = qrow(i, w);
    double init = 0.0;
    if (i < kQDiagSlots && g < nrow)
      init = Bin ? Bin[((int64_t)blockIdx.x * kQB + g) * kQB + c] : (g == c ? 1.0 : 0.0);
    x[i] = init;
  }
  __syncthreads();
  const int nref = nrow < kQB ? nrow : kQB;
  int buf = 0;
  for (int j = nref - 1; j >= 0; --j) {
    const double tj = tau_s[j];
    if (tj == 0.0) continue;  // uniform across the CTA
    double v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = vsm[qrow(i, w) * kQB + j];
#pragma unroll
    for (int i = 0; i < kQDiagSlots; ++i)
      if (qrow(i, w) == j) v[i] = 1.0;
    double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      p0 = fma(v[i], x[i], p0);
      p1 = fma(v[i + 1], x[i + 1], p1);
      p2 = fma(v[i + 2], x[i + 2], p2);
      p3 = fma(v[i + 3], x[i + 3], p3);
    }
    red[buf][w][c] = (p0 + p1) + (p2 + p3);
    __syncthreads();
    double wc = 0.0;
#pragma unroll
    for (int q = 0; q < kQWarps; ++q) wc += red[buf][q][c];
    wc *= tj;
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = fma(-v[i], wc, x[i]);
    buf ^= 1;
  }
  if (c < out_cols) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int g = qrow(i, w);
      if (g < nrow) Out[(c0 + g) * ldo + c] = x[i];
    }
  }
}

// make diag(R) >= 0: flip column j of Q and row j of R when R_jj < 0.  The
// signs are latched first (qr_diag_signs) because block 0 rewrites R_jj.
__global__ void qr_diag_signs(int cols, const double* R, int64_t ldr, int* flip) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < cols) flip[j] = R[(int64_t)j * ldr + j] < 0.0;
}

__global__ void qr_positive_diag(int64_t rows, int cols, double* Q, int64_t ldq, double* R,
                                 int64_t ldr, const int* flip) {
  const int j = blockIdx.y;
  if (!flip[j]) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x)
    Q[i * ldq + j] = -Q[i * ldq + j];
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < cols; c += blockDim.x)
      if (c >= j) R[(int64_t)j * ldr + c] = -R[(int64_t)j * ldr + c];
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

constexpr int kApplySmem = kQCH * kQB * (int)sizeof(double);

static int tsqr32(int64_t rows, int cols, const double* X, int64_t ldx, double* Q, int64_t ldq, double* R,
                  int64_t ldr, cudaStream_t s) {
  SPB_CUDA(cudaFuncSetAttribute(tsqr_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kApplySmem));
  Arena ar(s);
  struct Level {
    int64_t rows;
    int nch;
    double* V;
    double* tau;
    double* Rs;
  };
  std::vector<Level> lv;
  const double* in = X;
  int64_t in_ld = ldx;
  int in_cols = cols;
  int64_t r = rows;
  while (true) {
    Level L;
    L.rows = r;
    L.nch = ceil_div(r, kQCH);
    L.V = ar.alloc<double>((size_t)r * kQB);
    L.tau = ar.alloc<double>((size_t)L.nch * kQB);
    L.Rs = ar.alloc<double>((size_t)L.nch * kQB * kQB);
    if (!L.V || !L.tau || !L.Rs) {
      set_error("tsqr workspace allocation failed");
      return SP_ECUDA;
    }
    tsqr_leaf_kernel<<<L.nch, kQThreads, 0, s>>>(in, r, in_cols, in_ld, L.V, L.tau, L.Rs);
    count_launch();
    SPB_CHECK_LAUNCH();
    lv.push_back(L);
    if (L.nch == 1) break;
    in = L.Rs;
    in_ld = kQB;
    in_cols = kQB;
    r = (int64_t)L.nch * kQB;
  }
  copy_block<<<ceil_div((int64_t)cols * cols, 256), 256, 0, s>>>(cols, cols, lv.back().Rs, kQB, R, ldr);
  count_launch();
  SPB_CHECK_LAUNCH();
  const double* bin = nullptr;
  for (int l = (int)lv.size() - 1; l >= 0; --l) {
    const Level& L = lv[l];
    double* out;
    int64_t ldo;
    int oc;
    if (l == 0) {
      out = Q;
      ldo = ldq;
      oc = cols;
    } else {
      out = ar.alloc<double>((size_t)L.rows * kQB);
      if (!out) {
        set_error("tsqr workspace allocation failed");
        return SP_ECUDA;
      }
      ldo = kQB;
      oc = kQB;
    }
    tsqr_apply_kernel<<<L.nch, kQThreads, kApplySmem, s>>>(L.V, L.tau, L.rows, bin, out, ldo, oc);
    count_launch();
    SPB_CHECK_LAUNCH();
    bin = out;
  }
  int* flip = ar.alloc<int>((size_t)cols);
  if (!flip) {
    set_error("tsqr workspace allocation failed");
    return SP_ECUDA;
  }
  qr_diag_signs<<<ceil_div(cols, 64), 64, 0, s>>>(cols, R, ldr, flip);
  count_launch();
  SPB_CHECK_LAUNCH();
  dim3 g(std::min(ceil_div(rows, 256), 64), cols);
  qr_positive_diag<<<g, 256, 0, s>>>(rows, cols, Q, ldq, R, ldr, flip);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

// Wide inputs: 32-column panels, two block Gram-Schmidt passes against the
// previous panels, then a Householder TSQR of the projected panel.
int tsqr(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
         double* R, int64_t ldr, cudaStream_t s) {
  SPB_REQUIRE(cols >= 1 && rows >= cols, "tsqr needs rows >= cols >= 1");
  SPB_REQUIRE(ldx >= cols && ldq >= cols && ldr >= cols, "bad tsqr leading dimension");
  if (cols <= kQB) return tsqr32(rows, (int)cols, X, ldx, Q, ldq, R, ldr, s);
  SPB_CUDA(cudaMemset2DAsync(R, ldr * sizeof(double), 0, cols * sizeof(double), cols, s));
  Arena ar(s);
  SPB_ALLOC(ar, double, P, (size_t)rows * kQB);
  SPB_ALLOC(ar, double, T, (size_t)cols * kQB);
  for (int64_t p0 = 0; p0 < cols; p0 += kQB) {
    const int w = (int)std::min<int64_t>(kQB, cols - p0);
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
    SPB_TRY(tsqr32(rows, w, P, w, Q + p0, ldq, R + p0 * ldr + p0, ldr, s));
  }
  return SP_OK;
}

}  // namespace spb
