// K2: the single read of A.  Y (n x r) = A^T Z with Z (m x r), r <= 16.
//
// This is the reformulated form of the one-pass cross-Gramian products
// (src/svd.py:66 `gram += block.T @ out`, src/power.py:209-211
// `hc += block.T @ sub`): once the kept left basis Z = U_{C,r} of the sketch is
// known, A^T Z is everything the single-pass finalize needs from A
// ("algebra").  At r <= 16 it is HBM-bound on B200 (2r flop per
// 8-byte element against a ~5 flop/B FP64 ridge).
//
// Layout: A row-major, each thread owns V adjacent columns (one 16-byte load
// per row), a CTA of 256 threads covers 256*V columns.  Rows are split into
// S contiguous strips (grid.y) so the grid fills the 148 SMs; each CTA stages
// its strip of Z in shared memory (broadcast reads) and keeps the V x R
// accumulator tile in FP64 registers.  Strips are reduced in a fixed order by
// a second kernel, so results are bitwise reproducible.
#include "common.cuh"
#include "launch_count.cuh"

namespace spb {

int gemm(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
         cudaStream_t s);

constexpr int kSkThreads = 256;
constexpr int kSkZRows = 256;  // rows of Z staged per smem refill
constexpr int kSkUnroll = 4;   // rows whose loads are issued together

template <typename TA, int V>
struct VecLoad;
template <>
struct VecLoad<double, 2> {
  __device__ __forceinline__ static void load(const double* p, double (&o)[2]) {
    double2 v = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = v.x;
    o[1] = v.y;
  }
};
template <>
struct VecLoad<float, 4> {
  __device__ __forceinline__ static void load(const float* p, double (&o)[4]) {
    float4 v = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = v.x;
    o[1] = v.y;
    o[2] = v.z;
    o[3] = v.w;
  }
};

template <int R, typename TA, int V>
__global__ void __launch_bounds__(kSkThreads)
skinny_atz_kernel(const TA* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                  const double* __restrict__ Z, int64_t ldz, int64_t rows_per_split,
                  bool vec_ok, double* __restrict__ out, int64_t ldo, int64_t split_stride) {
  __shared__ __align__(16) double zs[kSkZRows * R];
  const int64_t j0 = ((int64_t)blockIdx.x * kSkThreads + threadIdx.x) * V;
  const int64_t rb = (int64_t)blockIdx.y * rows_per_split;
  const int64_t re = min(m, rb + rows_per_split);
  const bool active = j0 < n;
  const bool full = vec_ok && (j0 + V <= n);

  double acc[V][R];
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int c = 0; c < R; ++c) acc[v][c] = 0.0;

  for (int64_t base = rb; base < re; base += kSkZRows) {
    const int64_t left = re - base;
    const int cnt = left < kSkZRows ? (int)left : kSkZRows;
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * R; e += kSkThreads)
      zs[e] = Z[(base + e / R) * ldz + (e % R)];
    __syncthreads();
    if (!active) continue;
    const TA* arow = A + base * lda + j0;
    int i = 0;
    if (full) {
      for (; i + kSkUnroll <= cnt; i += kSkUnroll) {
        double a[kSkUnroll][V];
#pragma unroll
        for (int u = 0; u < kSkUnroll; ++u) VecLoad<TA, V>::load(arow + (int64_t)(i + u) * lda, a[u]);
#pragma unroll
        for (int u = 0; u < kSkUnroll; ++u) {
          const double* zr = zs + (i + u) * R;
#pragma unroll
          for (int c = 0; c < R; ++c) {
            const double zc = zr[c];
#pragma unroll
            for (int v = 0; v < V; ++v) acc[v][c] = fma(a[u][v], zc, acc[v][c]);
          }
        }
      }
    }
    for (; i < cnt; ++i) {
      double a[V];
#pragma unroll
      for (int v = 0; v < V; ++v) a[v] = (j0 + v < n) ? widen(__ldg(arow + (int64_t)i * lda + v)) : 0.0;
      const double* zr = zs + i * R;
#pragma unroll
      for (int c = 0; c < R; ++c)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v][c] = fma(a[v], zr[c], acc[v][c]);
    }
  }
  if (!active) return;
  double* o = out + (int64_t)blockIdx.y * split_stride;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    if (j0 + v < n) {
#pragma unroll
      for (int c = 0; c < R; ++c) o[(j0 + v) * ldo + c] = acc[v][c];
    }
  }
}

// Y[j, c] = sum_{s=0}^{S-1} P[s, j, c]  (fixed order)
__global__ void split_reduce_kernel(const double* __restrict__ P, int S, int64_t n, int r,
                                    double* __restrict__ Y, int64_t ldy) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * r) return;
  const int64_t j = e / r;
  const int c = (int)(e % r);
  double acc = 0.0;
  for (int s = 0; s < S; ++s) acc += P[(int64_t)s * n * r + e];
  Y[j * ldy + c] = acc;
}

template <int R, typename TA>
int skinny_tma_launch(const TA* A, int64_t m, int64_t n, int64_t lda, const double* Zc, double* Y, int64_t ldy,
                      cudaStream_t s);
bool skinny_tma_ok(const void* A, int a_dtype, int64_t n, int64_t lda);
int copy2d(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Y, int64_t ldy, cudaStream_t s);

template <int R, typename TA>
static int launch_skinny_r(const TA* A, int64_t m, int64_t n, int64_t lda, const double* Z,
                           int64_t ldz, double* Y, int64_t ldy, cudaStream_t s) {
  constexpr int V = sizeof(TA) == 8 ? 2 : 4;
  static const bool legacy = std::getenv("SPB_SKINNY_LEGACY") != nullptr;
  if (skinny_tma_ok(A, sizeof(TA) == 8 ? SP_F64 : SP_F32, n, lda) && m >= 1 && !legacy) {
    // TMA-streamed persistent path: Z packed contiguously (+ pad for the
    // 16-byte rounded bulk copy of the last row group)
    Arena ar(s);
    SPB_ALLOC(ar, double, Zc, (size_t)m * R + 2);
    SPB_TRY(copy2d(m, R, Z, ldz, Zc, R, s));
    return skinny_tma_launch<R, TA>(A, m, n, lda, Zc, Y, ldy, s);
  }
  const bool vec_ok = (lda % V == 0) && ((reinterpret_cast<uintptr_t>(A) % 16) == 0);
  const int gx = ceil_div(n, (int64_t)kSkThreads * V);
  // split rows so that ~6 CTAs per SM are in flight, with >= 64 rows per strip
  int S = std::max(1, std::min(ceil_div(6 * kNumSMs, gx), ceil_div(m, 64)));
  int64_t rps = ceil_div(m, S);
  S = ceil_div(m, rps);
  dim3 grid(gx, S);
  if (S == 1) {
    skinny_atz_kernel<R, TA, V><<<grid, kSkThreads, 0, s>>>(A, m, n, lda, Z, ldz, rps, vec_ok, Y, ldy, 0);
    count_launch();
    SPB_CHECK_LAUNCH();
    return SP_OK;
  }
  Arena ar(s);
  SPB_ALLOC(ar, double, part, (size_t)S * n * R);
  skinny_atz_kernel<R, TA, V><<<grid, kSkThreads, 0, s>>>(A, m, n, lda, Z, ldz, rps, vec_ok, part, R, n * R);
  count_launch();
  SPB_CHECK_LAUNCH();
  split_reduce_kernel<<<ceil_div(n * R, 256), 256, 0, s>>>(part, S, n, R, Y, ldy);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

template <typename TA>
static int dispatch_skinny(int r, const TA* A, int64_t m, int64_t n, int64_t lda, const double* Z,
                           int64_t ldz, double* Y, int64_t ldy, cudaStream_t s) {
  switch (r) {
#define SPB_R(RR) \
  case RR:        \
    return launch_skinny_r<RR, TA>(A, m, n, lda, Z, ldz, Y, ldy, s);
    SPB_R(1) SPB_R(2) SPB_R(3) SPB_R(4) SPB_R(5) SPB_R(6) SPB_R(7) SPB_R(8)
    SPB_R(9) SPB_R(10) SPB_R(11) SPB_R(12) SPB_R(13) SPB_R(14) SPB_R(15) SPB_R(16)
#undef SPB_R
  }
  set_error("skinny A^T Z supports r <= 16");
  return SP_ECONFIG;
}

int skinny_atz(const void* A, int a_dtype, int64_t m, int64_t n, int64_t lda, const double* Z,
               int64_t ldz, int r, double* Y, int64_t ldy, cudaStream_t s) {
  SPB_REQUIRE(r >= 1 && lda >= n && ldz >= r && ldy >= r, "bad skinny shapes");
  if (n == 0) return SP_OK;
  if (m == 0) {
    SPB_CUDA(cudaMemset2DAsync(Y, ldy * sizeof(double), 0, r * sizeof(double), n, s));
    return SP_OK;
  }
  if (r <= 16) {
    if (a_dtype == SP_F64) return dispatch_skinny<double>(r, (const double*)A, m, n, lda, Z, ldz, Y, ldy, s);
    if (a_dtype == SP_F32) return dispatch_skinny<float>(r, (const float*)A, m, n, lda, Z, ldz, Y, ldy, s);
    set_error("unknown dtype tag");
    return SP_ECONFIG;
  }
  if (a_dtype == SP_F32) {
    // FP32-stored A: 16-column slabs of Z, one read of A per slab
    for (int c0 = 0; c0 < r; c0 += 16) {
      const int w = std::min(16, r - c0);
      SPB_TRY(dispatch_skinny<float>(w, (const float*)A, m, n, lda, Z + c0, ldz, Y + c0, ldy, s));
    }
    return SP_OK;
  }
  // wide right-hand side: compute-bound, use the DMMA GEMM (Y = A^T Z)
  return gemm(1, 0, n, r, m, 1.0, (const double*)A, lda, Z, ldz, 0.0, Y, ldy, s);
}

}  // namespace spb
