// K4: Householder TSQR for tall-skinny matrices (cols <= 32 per panel).
//
// Replaces thin_qr / np.linalg.qr (src/kernels.py:74-84) on the path.  The
// sketch bases on this path are numerically rank deficient (SURVEY.md 7 "Hard
// parts"): CholeskyQR2 breaks down, so orthogonalisation is Householder
// based, which keeps the span of every direction to eps * ||X|| regardless of
// conditioning.
//
// Tree: level 0 splits the rows into chunks of CH = 256 * (32 / B) rows; one
// CTA factors a chunk with each thread holding 32/B rows of the chunk in
// registers (B doubles per row).  Column dot products are reduced with a warp
// reduce-scatter (log2(B) shuffle rounds, one column per lane) and a fixed
// order sum over the 8 warps, so the result is bitwise reproducible.  The
// B x B R factors are stacked and factored again until one chunk remains.
// Q is then formed top-down by applying each chunk's reflectors to its block
// of the parent Q.
#include "common.cuh"
#include "launch_count.cuh"

#include <vector>

namespace spb {

int gemm(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
         cudaStream_t s);

constexpr int kQrThreads = 256;
constexpr int kQrWarps = kQrThreads / 32;

template <int B>
struct QrShape {
  static constexpr int RPT = 32 / B;             // rows per thread
  static constexpr int CH = kQrThreads * RPT;    // rows per chunk
};

// Reduce p[0..B) over the 256 threads of the CTA; on return every thread sees
// out_s[c] = scale * sum over rows.  Deterministic order.
template <int B>
__device__ __forceinline__ void block_reduce_cols(double (&p)[B], double* red /*[kQrWarps][B]*/,
                                                  double* out_s /*[B]*/, double scale) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // reduce-scatter: after log2(B) rounds lane holds column col(lane)
  int col = 0;
#pragma unroll
  for (int half = B / 2, off = 16; half >= 1; half >>= 1, off >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = upper ? p[i] : p[i + half];
      const double keep = upper ? p[i + half] : p[i];
      p[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
    if (upper) col += half;
  }
  // remaining butterfly rounds when B < 32
  constexpr int kLanesPerCol = 32 / B;
#pragma unroll
  for (int off = kLanesPerCol / 2; off >= 1; off >>= 1) p[0] += __shfl_xor_sync(0xffffffffu, p[0], off);
  if ((lane % kLanesPerCol) == 0) red[warp * B + col] = p[0];
  __syncthreads();
  if (threadIdx.x < B) {
    double acc = 0.0;
#pragma unroll
    for (int w = 0; w < kQrWarps; ++w) acc += red[w * B + threadIdx.x];
    out_s[threadIdx.x] = acc * scale;
  }
  __syncthreads();
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double acc = 0.0;
#pragma unroll
  for (int w = 0; w < kQrWarps; ++w) acc += red[w];
  __syncthreads();
  return acc;
}

// Factor chunk blockIdx.x of X (rows x cols, cols <= B).  Writes reflectors
// (strictly below the diagonal of each chunk) to V (rows x B, ld B), tau to
// tau[chunk*B + j] and the chunk's upper-trapezoidal R into
// Rs[chunk*B .. chunk*B+B) x B (zero padded).
template <int B>
__global__ void __launch_bounds__(kQrThreads, 1)
tsqr_leaf_kernel(const double* __restrict__ X, int64_t rows, int cols, int64_t ldx,
                 double* __restrict__ V, double* __restrict__ tau, double* __restrict__ Rs) {
  constexpr int RPT = QrShape<B>::RPT, CH = QrShape<B>::CH;
  __shared__ double red[kQrWarps * B];
  __shared__ double wsum[B];
  __shared__ double scal[2];
  const int64_t c0 = (int64_t)blockIdx.x * CH;
  const int64_t left = rows - c0;
  const int nrow = left < CH ? (int)left : CH;
  double x[RPT][B];
#pragma unroll
  for (int e = 0; e < RPT; ++e) {
    const int lr = e * kQrThreads + threadIdx.x;
#pragma unroll
    for (int c = 0; c < B; ++c)
      x[e][c] = (lr < nrow && c < cols) ? X[(c0 + lr) * ldx + c] : 0.0;
  }
  const int nref = min(nrow, B);
  for (int j = 0; j < nref; ++j) {
    // column j: diagonal element and squared norm below it
    double sq = 0.0;
#pragma unroll
    for (int e = 0; e < RPT; ++e) {
      const int lr = e * kQrThreads + threadIdx.x;
      double xj = 0.0;
#pragma unroll
      for (int c = 0; c < B; ++c) xj = (c == j) ? x[e][c] : xj;
      if (lr > j && lr < nrow) sq = fma(xj, xj, sq);
      if (lr == j) scal[0] = xj;
    }
    const double sigma2 = block_sum(sq, red);  // contains the sync that publishes scal[0]
    const double alpha = scal[0];
    double beta = alpha, tj = 0.0, inv = 0.0;
    if (sigma2 > 0.0) {
      const double nrm = sqrt(fma(alpha, alpha, sigma2));
      beta = alpha >= 0.0 ? -nrm : nrm;
      tj = (beta - alpha) / beta;
      inv = 1.0 / (alpha - beta);
    }
    // v (unit diagonal) and partial dots w_c = sum v_i x_ic for c > j
    double vv[RPT];
    double p[B];
#pragma unroll
    for (int c = 0; c < B; ++c) p[c] = 0.0;
#pragma unroll
    for (int e = 0; e < RPT; ++e) {
      const int lr = e * kQrThreads + threadIdx.x;
      double xj = 0.0;
#pragma unroll
      for (int c = 0; c < B; ++c) xj = (c == j) ? x[e][c] : xj;
      vv[e] = (lr == j) ? 1.0 : ((lr > j && lr < nrow) ? xj * inv : 0.0);
#pragma unroll
      for (int c = 0; c < B; ++c) p[c] = (c > j) ? fma(vv[e], x[e][c], p[c]) : p[c];
    }
    block_reduce_cols<B>(p, red, wsum, tj);
#pragma unroll
    for (int e = 0; e < RPT; ++e) {
      const int lr = e * kQrThreads + threadIdx.x;
#pragma unroll
      for (int c = 0; c < B; ++c) {
        if (c > j) x[e][c] = fma(-vv[e], wsum[c], x[e][c]);
        if (c == j) x[e][c] = (lr == j) ? beta : ((lr > j) ? vv[e] : x[e][c]);
      }
    }
    if (threadIdx.x == 0) tau[(int64_t)blockIdx.x * B + j] = tj;
  }
  if (threadIdx.x < B && threadIdx.x >= nref) tau[(int64_t)blockIdx.x * B + threadIdx.x] = 0.0;
#pragma unroll
  for (int e = 0; e < RPT; ++e) {
    const int lr = e * kQrThreads + threadIdx.x;
    if (lr < nrow) {
#pragma unroll
      for (int c = 0; c < B; ++c) V[(c0 + lr) * B + c] = (lr > c) ? x[e][c] : 0.0;
    }
    if (lr < B) {
#pragma unroll
      for (int c = 0; c < B; ++c)
        Rs[((int64_t)blockIdx.x * B + lr) * B + c] = (lr < nrow && c >= lr) ? x[e][c] : 0.0;
    }
  }
}

// Out rows of chunk blockIdx.x = H_0 ... H_{B-1} [Bin_chunk ; 0], where
// Bin_chunk = Bin[chunk*B .. +B) (ld B), or the identity when Bin == nullptr.
template <int B>
__global__ void __launch_bounds__(kQrThreads, 1)
tsqr_apply_kernel(const double* __restrict__ V, const double* __restrict__ tau, int64_t rows,
                  const double* __restrict__ Bin, double* __restrict__ Out, int64_t ldo,
                  int out_cols) {
  constexpr int RPT = QrShape<B>::RPT, CH = QrShape<B>::CH;
  __shared__ double red[kQrWarps * B];
  __shared__ double wsum[B];
  const int64_t c0 = (int64_t)blockIdx.x * CH;
  const int64_t left = rows - c0;
  const int nrow = left < CH ? (int)left : CH;
  double w[RPT][B], v[RPT][B];
#pragma unroll
  for (int e = 0; e < RPT; ++e) {
    const int lr = e * kQrThreads + threadIdx.x;
#pragma unroll
    for (int c = 0; c < B; ++c) {
      v[e][c] = (lr < nrow) ? V[(c0 + lr) * B + c] : 0.0;
      double init = 0.0;
      if (lr < B && lr < nrow) init = Bin ? Bin[((int64_t)blockIdx.x * B + lr) * B + c] : (lr == c ? 1.0 : 0.0);
      w[e][c] = init;
    }
  }
  const int nref = min(nrow, B);
  for (int j = nref - 1; j >= 0; --j) {
    const double tj = tau[(int64_t)blockIdx.x * B + j];
    if (tj == 0.0) continue;  // uniform across the CTA
    double p[B];
    double vj[RPT];
#pragma unroll
    for (int c = 0; c < B; ++c) p[c] = 0.0;
#pragma unroll
    for (int e = 0; e < RPT; ++e) {
      const int lr = e * kQrThreads + threadIdx.x;
      double vs = 0.0;
#pragma unroll
      for (int c = 0; c < B; ++c) vs = (c == j) ? v[e][c] : vs;
      vj[e] = (lr == j) ? 1.0 : ((lr > j && lr < nrow) ? vs : 0.0);
#pragma unroll
      for (int c = 0; c < B; ++c) p[c] = fma(vj[e], w[e][c], p[c]);
    }
    block_reduce_cols<B>(p, red, wsum, tj);
#pragma unroll
    for (int e = 0; e < RPT; ++e)
#pragma unroll
      for (int c = 0; c < B; ++c) w[e][c] = fma(-vj[e], wsum[c], w[e][c]);
  }
#pragma unroll
  for (int e = 0; e < RPT; ++e) {
    const int lr = e * kQrThreads + threadIdx.x;
    if (lr < nrow) {
#pragma unroll
      for (int c = 0; c < B; ++c)
        if (c < out_cols) Out[(c0 + lr) * ldo + c] = w[e][c];
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

template <int B>
static int tsqr_panel(int64_t rows, int cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
                      double* R, int64_t ldr, cudaStream_t s) {
  constexpr int CH = QrShape<B>::CH;
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
    L.nch = ceil_div(r, CH);
    L.V = ar.alloc<double>((size_t)r * B);
    L.tau = ar.alloc<double>((size_t)L.nch * B);
    L.Rs = ar.alloc<double>((size_t)L.nch * B * B);
    if (!L.V || !L.tau || !L.Rs) {
      set_error("tsqr workspace allocation failed");
      return SP_ECUDA;
    }
    tsqr_leaf_kernel<B><<<L.nch, kQrThreads, 0, s>>>(in, r, in_cols, in_ld, L.V, L.tau, L.Rs);
    count_launch();
    SPB_CHECK_LAUNCH();
    lv.push_back(L);
    if (L.nch == 1) break;
    in = L.Rs;
    in_ld = B;
    in_cols = B;
    r = (int64_t)L.nch * B;
  }
  // R = top-level R (B x B), keep cols x cols
  copy_block<<<ceil_div((int64_t)cols * cols, 256), 256, 0, s>>>(cols, cols, lv.back().Rs, B, R, ldr);
  count_launch();
  SPB_CHECK_LAUNCH();
  // Q top-down
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
      out = ar.alloc<double>((size_t)L.rows * B);
      if (!out) {
        set_error("tsqr workspace allocation failed");
        return SP_ECUDA;
      }
      ldo = B;
      oc = B;
    }
    tsqr_apply_kernel<B><<<L.nch, kQrThreads, 0, s>>>(L.V, L.tau, L.rows, bin, out, ldo, oc);
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

static int tsqr32(int64_t rows, int cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
                  double* R, int64_t ldr, cudaStream_t s) {
  if (cols <= 8) return tsqr_panel<8>(rows, cols, X, ldx, Q, ldq, R, ldr, s);
  if (cols <= 16) return tsqr_panel<16>(rows, cols, X, ldx, Q, ldq, R, ldr, s);
  return tsqr_panel<32>(rows, cols, X, ldx, Q, ldq, R, ldr, s);
}

// Wide inputs: 32-column panels, two block Gram-Schmidt passes against the
// previous panels, then a Householder TSQR of the projected panel.
int tsqr(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
         double* R, int64_t ldr, cudaStream_t s) {
  SPB_REQUIRE(cols >= 1 && rows >= cols, "tsqr needs rows >= cols >= 1");
  SPB_REQUIRE(ldx >= cols && ldq >= cols && ldr >= cols, "bad tsqr leading dimension");
  if (cols <= 32) return tsqr32(rows, (int)cols, X, ldx, Q, ldq, R, ldr, s);
  SPB_CUDA(cudaMemset2DAsync(R, ldr * sizeof(double), 0, cols * sizeof(double), cols, s));
  Arena ar(s);
  SPB_ALLOC(ar, double, P, (size_t)rows * 32);
  SPB_ALLOC(ar, double, T, (size_t)cols * 32);
  for (int64_t p0 = 0; p0 < cols; p0 += 32) {
    const int w = (int)std::min<int64_t>(32, cols - p0);
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
