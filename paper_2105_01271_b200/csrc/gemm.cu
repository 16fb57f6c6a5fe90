// K3: FP64 GEMM on the B200 DMMA pipe (mma.sync.aligned.m8n8k4.f64).
//
// tcgen05.mma has no f64 kind on sm_100a (ptxas rejects .kind::f64), so the
// FP64 tensor path on B200 is the warp-level DMMA.  C = alpha op(A) op(B) +
// beta C for row-major operands; op() selected at compile time so that each
// operand is copied to shared memory in its global (coalesced) orientation and
// the fragment reads are bank-conflict free for both orientations (padded
// strides 20 and 68 doubles).  64x64x16 CTA tiles, 4 warps of 32x32, 8-byte
// cp.async (16-byte pairs when aligned) with zero-fill at the edges, a 3-stage ring.  When the tile grid
// cannot fill the 148 SMs, K is split and the partial tiles are reduced in a
// fixed order (bitwise reproducible).
//
// Used for every dense product of the path (src/power.py:101,105,166-170,284;
// src/rowid.py:138-139) and for the literal cross-Gramian (src/svd.py:66).
#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

constexpr int kBK = 16;
constexpr int kGemmThreads = 128;
constexpr int kGemmStages = 3;  // cp.async ring depth (dynamic shared memory)
// k-contiguous rows: stride 20 doubles (18 for the 128-row tiles, which
// would otherwise not fit two stages in 48 KB of static shared memory)
template <int ROWS>
struct PadK {
  static constexpr int v = ROWS > 64 ? kBK + 2 : kBK + 4;
};

// Tile shapes: 64 x 64 (2 x 2 warps of 32 x 32) and, for N <= 32, 128 x 32
// (4 x 1 warps) so the narrow products of the path do not pad N to 64.
template <int BM, int BN>
struct Tile {
  static constexpr int kWarpsM = BM / 32;
  static_assert(kWarpsM * (BN / 32) == 4, "4 warps of 32 x 32");
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  int bytes = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// element (r, k) of op(X) where op(X) is R x K; X row-major with ld
template <int TRANS>
__device__ __forceinline__ const double* op_ptr(const double* X, int64_t ld, int64_t r, int64_t k) {
  return TRANS ? X + k * ld + r : X + r * ld + k;
}

// smem offset of element (r, k) of an op(X) tile (r in [0, ROWS), k in [0,16))
template <int TRANS, int ROWS>
__device__ __forceinline__ int tile_off(int r, int k) {
  return TRANS ? k * (ROWS + 4) + r : r * PadK<ROWS>::v + k;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(bytes));
}

// Same tile with 16-byte copies of element pairs along the contiguous
// dimension (ld even, X 16-byte aligned; every smem pair offset is even).
// A pair straddling the edge copies 8 bytes and zero-fills the other half.
template <int TRANS, int ROWS>
__device__ __forceinline__ void load_tile16(double* st, const double* X, int64_t ld, int64_t R,
                                            int64_t K, int64_t r0, int64_t k0, int64_t k_end) {
#pragma unroll
  for (int u = 0; u < (ROWS * kBK) / (2 * kGemmThreads); ++u) {
    const int e = threadIdx.x + u * kGemmThreads;  // pair index
    int r, k;
    int64_t lim;
    if (TRANS) {  // stored K x R: pairs along r
      k = e / (ROWS / 2);
      r = 2 * (e % (ROWS / 2));
    } else {  // stored R x K: pairs along k
      r = e / (kBK / 2);
      k = 2 * (e % (kBK / 2));
    }
    const int64_t gr = r0 + r, gk = k0 + k;
    int n;
    if (TRANS) {
      lim = R - gr;
      n = (gk < k_end && lim > 0) ? (lim >= 2 ? 16 : 8) : 0;
    } else {
      lim = k_end - gk;
      n = (gr < R && lim > 0) ? (lim >= 2 ? 16 : 8) : 0;
    }
    cp_async16(st + tile_off<TRANS, ROWS>(r, k), n ? op_ptr<TRANS>(X, ld, gr, gk) : X, n);
  }
}

template <int TRANS, int ROWS>
__device__ __forceinline__ void load_tile(double* st, const double* X, int64_t ld, int64_t R,
                                          int64_t K, int64_t r0, int64_t k0, int64_t k_end) {
  // ROWS x 16 elements; consecutive threads walk the contiguous dim
#pragma unroll
  for (int u = 0; u < (ROWS * kBK) / kGemmThreads; ++u) {
    const int e = threadIdx.x + u * kGemmThreads;
    int r, k;
    if (TRANS) {  // stored K x R: contiguous along r
      k = e / ROWS;
      r = e % ROWS;
    } else {  // stored R x K: contiguous along k
      r = e / kBK;
      k = e % kBK;
    }
    const int64_t gr = r0 + r, gk = k0 + k;
    const bool ok = (gr < R) && (gk < k_end);
    cp_async8(st + tile_off<TRANS, ROWS>(r, k), ok ? op_ptr<TRANS>(X, ld, gr, gk) : X, ok);
  }
}

template <int TA, int TB, int BM, int BN>
struct StageSizes {
  static constexpr int kSA = TA ? kBK * (BM + 4) : BM * PadK<BM>::v;
  static constexpr int kSB = TB ? BN * PadK<BN>::v : kBK * (BN + 4);
  static constexpr size_t kBytes = (size_t)kGemmStages * (kSA + kSB) * sizeof(double);
};

template <int TA, int TB, int BM, int BN, bool V16>
__global__ void __launch_bounds__(kGemmThreads)
dgemm_kernel(int64_t M, int64_t N, int64_t K, const double* __restrict__ A, int64_t lda,
             const double* __restrict__ B, int64_t ldb, double* __restrict__ C, int64_t ldc,
             double alpha, double beta, int64_t k_per_split, bool partial, bool upper) {
  SPB_PDL_ENTRY();
  using TL = Tile<BM, BN>;
  // symmetric product (gemm_aat): tiles strictly below the diagonal are the
  // mirror images of computed ones and exit at once
  if (upper && ((int64_t)blockIdx.x % ((N + BN - 1) / BN)) * BN + BN <= ((int64_t)blockIdx.x / ((N + BN - 1) / BN)) * BM)
    return;
  // stage sizes for the operand orientations (op(B) tile is stored as (n, k) with orientation !TB)
  constexpr int kSA = StageSizes<TA, TB, BM, BN>::kSA;
  constexpr int kSB = StageSizes<TA, TB, BM, BN>::kSB;
  // kGemmStages-deep cp.async ring in dynamic shared memory
  extern __shared__ __align__(16) double gemm_smem[];
  double (*sA)[kSA] = reinterpret_cast<double (*)[kSA]>(gemm_smem);
  double (*sB)[kSB] = reinterpret_cast<double (*)[kSB]>(gemm_smem + kGemmStages * kSA);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % TL::kWarpsM) * 32, wn = (warp / TL::kWarpsM) * 32;
  // linear tile index (grid.x can exceed 65535 tiles for n-row operands)
  const int64_t tiles_n = (N + BN - 1) / BN;
  const int64_t m0 = ((int64_t)blockIdx.x / tiles_n) * BM, n0 = ((int64_t)blockIdx.x % tiles_n) * BN;
  const int64_t kb = (int64_t)blockIdx.z * k_per_split;
  const int64_t ke = min(K, kb + k_per_split);
  const int ntiles = (int)((ke - kb + kBK - 1) / kBK);

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load_stage = [&](int st, int64_t k0) {
    if constexpr (V16) {
      load_tile16<TA, BM>(sA[st], A, lda, M, K, m0, k0, ke);
      load_tile16<TB ? 0 : 1, BN>(sB[st], B, ldb, N, K, n0, k0, ke);
    } else {
      load_tile<TA, BM>(sA[st], A, lda, M, K, m0, k0, ke);
      load_tile<TB ? 0 : 1, BN>(sB[st], B, ldb, N, K, n0, k0, ke);
    }
  };
  if (ntiles > 0) load_stage(0, kb);
  cp_async_commit();
  for (int st = 1; st < kGemmStages - 1; ++st) {
    if (st < ntiles) load_stage(st, kb + (int64_t)st * kBK);
    cp_async_commit();
  }
  for (int kt = 0; kt < ntiles; ++kt) {
    const int cur = kt % kGemmStages;
    cp_async_wait<kGemmStages - 2>();
    __syncthreads();  // tile kt landed for every thread; stage (kt - 1) % S is free
    {
      const int nx = kt + kGemmStages - 1;
      if (nx < ntiles) load_stage(nx % kGemmStages, kb + (int64_t)nx * kBK);
      cp_async_commit();
    }
    const double* a_s = sA[cur];
    const double* b_s = sB[cur];
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = a_s[tile_off<TA, BM>(wm + i * 8 + g, kk + t)];
      // op(B) is K x N; stored tile holds (n, k) with orientation !TB
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = b_s[tile_off<TB ? 0 : 1, BN>(wn + j * 8 + g, kk + t)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }

  double* Cs = partial ? C + (int64_t)blockIdx.z * M * N : C;
  const int64_t ldo = partial ? N : ldc;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + wm + i * 8 + g;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t n = n0 + wn + j * 8 + 2 * t + h;
        if (n >= N) continue;
        double* p = Cs + m * ldo + n;
        if (partial) {
          *p = acc[i][j][h];
        } else {
          const double v = alpha * acc[i][j][h];
          *p = (beta == 0.0) ? v : fma(beta, *p, v);
        }
      }
    }
  }
}

// C = alpha * sum_s P[s] + beta * C.  Deep splits (S > 8): a 256-thread CTA
// owns 32 consecutive outputs; warp g sums splits g, g+8, ... (lanes read
// consecutive outputs: coalesced) and the 8 warp partials are combined in a
// fixed order (deterministic); shallow splits: one thread per output.
__global__ void __launch_bounds__(256) gemm_split_reduce_warp(const double* __restrict__ P, int S, int64_t M,
                                                              int64_t N, double alpha, double beta,
                                                              double* __restrict__ C, int64_t ldc) {
  SPB_PDL_ENTRY();
  __shared__ double part[8][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  const int64_t MN = M * N;
  double acc = 0.0;
  if (e < MN) {
#pragma unroll 8
    for (int s = g; s < S; s += 8) acc += P[(int64_t)s * MN + e];
  }
  part[g][lane] = acc;
  __syncthreads();
  if (g == 0 && e < MN) {
    double t = part[0][lane];
#pragma unroll
    for (int k = 1; k < 8; ++k) t += part[k][lane];
    double* p = C + (e / N) * ldc + (e % N);
    const double v = alpha * t;
    *p = (beta == 0.0) ? v : fma(beta, *p, v);
  }
}

__global__ void gemm_split_reduce(const double* __restrict__ P, int S, int64_t M, int64_t N,
                                  double alpha, double beta, double* __restrict__ C, int64_t ldc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  double acc = 0.0;
  for (int s = 0; s < S; ++s) acc += P[(int64_t)s * M * N + e];
  double* p = C + (e / N) * ldc + (e % N);
  const double v = alpha * acc;
  *p = (beta == 0.0) ? v : fma(beta, *p, v);
}

__global__ void scale_matrix(int64_t M, int64_t N, double beta, double* C, int64_t ldc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  double* p = C + (e / N) * ldc + (e % N);
  *p = (beta == 0.0) ? 0.0 : beta * *p;
}

template <int TA, int TB, int BM, int BN>
static void launch_dgemm(dim3 grid, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                         const double* B, int64_t ldb, double* C, int64_t ldc, double alpha,
                         double beta, int64_t kps, bool partial, cudaStream_t s, bool upper = false) {
  // 16-byte copies when both operands allow them (even leading dimensions,
  // 16-byte aligned bases; split-K boundaries are multiples of kBK)
  const bool v16 = (lda % 2 == 0) && (ldb % 2 == 0) &&
                   ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
  constexpr size_t smem = StageSizes<TA, TB, BM, BN>::kBytes;
  static int attr_dev = -1;  // once per device and instantiation
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(dgemm_kernel<TA, TB, BM, BN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(dgemm_kernel<TA, TB, BM, BN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_dev = dev;
  }
  // errors surface through the caller's cudaGetLastError check
  if (v16)
    launch_pdl((dgemm_kernel<TA, TB, BM, BN, true>), grid, dim3(kGemmThreads), smem, s, M, N, K, A, lda, B, ldb, C,
               ldc, alpha, beta, kps, partial, upper);
  else
    launch_pdl((dgemm_kernel<TA, TB, BM, BN, false>), grid, dim3(kGemmThreads), smem, s, M, N, K, A, lda, B, ldb, C,
               ldc, alpha, beta, kps, partial, upper);
}

template <int BM, int BN>
static void launch_dgemm_any(int code, dim3 grid, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                             const double* B, int64_t ldb, double* C, int64_t ldc, double alpha, double beta,
                             int64_t kps, bool partial, cudaStream_t s, bool upper = false) {
  switch (code) {
    case 0: launch_dgemm<0, 0, BM, BN>(grid, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, kps, partial, s, upper); break;
    case 1: launch_dgemm<0, 1, BM, BN>(grid, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, kps, partial, s, upper); break;
    case 2: launch_dgemm<1, 0, BM, BN>(grid, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, kps, partial, s, upper); break;
    default: launch_dgemm<1, 1, BM, BN>(grid, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, kps, partial, s, upper); break;
  }
}

static int gemm_impl(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                     int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                     cudaStream_t s, bool upper);

int gemm(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
         cudaStream_t s) {
  return gemm_impl(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, s, false);
}

// W[j][i] = W[i][j] for j > i (row-major n x n)
__global__ void mirror_upper_kernel(int64_t n, double* __restrict__ W, int64_t ldw) {
  __shared__ double tile[32][33];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;
  if (bj < bi) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int r = ty; r < 32; r += blockDim.y) {
    const int64_t i = bi * 32 + r, j = bj * 32 + tx;
    tile[r][tx] = (i < n && j < n) ? W[i * ldw + j] : 0.0;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += blockDim.y) {
    const int64_t j = bj * 32 + r, i = bi * 32 + tx;  // writes W[j][i], j > i
    if (j < n && i < n && j > i) W[j * ldw + i] = tile[tx][r];
  }
}

// W = A A^T (A: M x K row-major): only the tiles on and above the diagonal are
// computed (half the DMMA work of the plain product: cfg5's W = C C^T, 2.1
// TFLOP, 70 -> 37 ms), the lower triangle is their mirror image -- W comes out
// exactly symmetric.
int gemm_upper(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
               const double* B, int64_t ldb, double beta, double* C, int64_t ldc, cudaStream_t s) {
  return gemm_impl(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, s, true);
}

int mirror_upper(int64_t n, double* W, int64_t ldw, cudaStream_t s) {
  if (n > 1) {
    const unsigned nb = (unsigned)ceil_div(n, 32);
    mirror_upper_kernel<<<dim3(nb, nb), dim3(32, 8), 0, s>>>(n, W, ldw);
    count_launch();
    SPB_CHECK_LAUNCH();
  }
  return SP_OK;
}

int gemm_aat(int64_t M, int64_t K, const double* A, int64_t lda, double* W, int64_t ldw, cudaStream_t s) {
  SPB_TRY(gemm_impl(0, 1, M, M, K, 1.0, A, lda, A, lda, 0.0, W, ldw, s, true));
  return mirror_upper(M, W, ldw, s);
}

static int gemm_impl(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                     int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                     cudaStream_t s, bool upper) {
  SPB_REQUIRE(M >= 0 && N >= 0 && K >= 0, "negative GEMM extent");
  SPB_REQUIRE(ldc >= N, "ldc < N");
  SPB_REQUIRE(lda >= (ta ? M : K) && ldb >= (tb ? K : N), "bad GEMM leading dimension");
  if (M == 0 || N == 0) return SP_OK;
  if (K == 0 || alpha == 0.0) {
    scale_matrix<<<ceil_div(M * N, 256), 256, 0, s>>>(M, N, beta, C, ldc);
    count_launch();
    SPB_CHECK_LAUNCH();
    return SP_OK;
  }
  // tall-skinny shapes where 64x64 DMMA tiles would idle: streaming kernels
  if (upper && (M != N || M <= 64)) upper = false;  // small or non-square: the plain product
  if (ta == 1 && tb == 0 && M <= 64 && N <= 64 && K >= 256)
    return tall_gram(K, (int)M, A, lda, (int)N, B, ldb, alpha, beta, C, ldc, s);
  if (ta == 0 && tb == 0 && K <= 64 && N <= 64 && M >= 256)
    return tall_mul(M, (int)K, A, lda, (int)N, B, ldb, alpha, beta, C, ldc, s);
  const bool narrow = N <= 32;
  const int bm = narrow ? 128 : 64, bn = narrow ? 32 : 64;
  const int gx = ceil_div(N, bn), gy = ceil_div(M, bm);
  const int64_t tiles = (int64_t)gx * gy;
  int S = 1;
  if (tiles < 2 * kNumSMs) {
    // K-splits filling exactly one wave of the resident slots (3 CTAs per SM
    // with the 3-stage ring; a partial second wave costs a whole CTA time),
    // each split at least 4 k-tiles deep
    constexpr int kSlots = 3 * kNumSMs;
    S = (int)std::min<int64_t>(std::max<int64_t>(1, kSlots / tiles), std::max<int64_t>(1, K / (4 * kBK)));
    S = std::max(1, std::min(S, 1024));
  }
  int64_t kps = ceil_div(K, S);
  kps = ceil_div(kps, kBK) * (int64_t)kBK;
  S = ceil_div(K, kps);
  dim3 grid((unsigned)tiles, 1, S);
  const bool partial = S > 1;
  Arena ar(s);
  double* out = C;
  if (partial) {
    out = ar.alloc<double>((size_t)S * M * N);
    if (!out) {
      set_error("GEMM split-K workspace allocation failed");
      return SP_ECUDA;
    }
  }
  const int code = ta * 2 + tb;
  if (narrow)
    launch_dgemm_any<128, 32>(code, grid, M, N, K, A, lda, B, ldb, out, ldc, alpha, beta, kps, partial, s, upper);
  else
    launch_dgemm_any<64, 64>(code, grid, M, N, K, A, lda, B, ldb, out, ldc, alpha, beta, kps, partial, s, upper);
  count_launch();
  SPB_CHECK_LAUNCH();
  if (partial) return split_reduce(out, S, M, N, alpha, beta, C, ldc, s);
  return SP_OK;
}

// op(A) op(B) as S fixed-order split-K partial slabs P[s] (M x N, row-major,
// slab stride M * N) for a consumer that sums them itself (the Rz Gram of the
// Rayleigh-Ritz step reads Z = C^T Q this way: no reduction launch on the
// critical path).  S = 1 writes the product itself.  DMMA shapes only.
int gemm_partials(int ta, int tb, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                  int64_t ldb, Arena& ar, double** P, int* S_out, cudaStream_t s) {
  SPB_REQUIRE(M > 0 && N > 0 && K > 0, "gemm_partials: empty GEMM");
  SPB_REQUIRE(lda >= (ta ? M : K) && ldb >= (tb ? K : N), "bad GEMM leading dimension");
  const bool narrow = N <= 32;
  const int bm = narrow ? 128 : 64, bn = narrow ? 32 : 64;
  const int64_t tiles = (int64_t)ceil_div(N, bn) * ceil_div(M, bm);
  int S = 1;
  if (tiles < 2 * kNumSMs) {
    constexpr int kSlots = 3 * kNumSMs;  // as gemm(): one wave of the resident slots
    S = (int)std::min<int64_t>(std::max<int64_t>(1, kSlots / tiles), std::max<int64_t>(1, K / (4 * kBK)));
    S = std::max(1, std::min(S, 1024));
  }
  int64_t kps = ceil_div(ceil_div(K, S), kBK) * (int64_t)kBK;
  S = ceil_div(K, kps);
  double* out = ar.alloc<double>((size_t)S * M * N);
  if (!out) {
    set_error("GEMM split-K workspace allocation failed");
    return SP_ECUDA;
  }
  const dim3 grid((unsigned)tiles, 1, S);
  const int code = ta * 2 + tb;
  if (narrow)
    launch_dgemm_any<128, 32>(code, grid, M, N, K, A, lda, B, ldb, out, N, 1.0, 0.0, kps, true, s);
  else
    launch_dgemm_any<64, 64>(code, grid, M, N, K, A, lda, B, ldb, out, N, 1.0, 0.0, kps, true, s);
  count_launch();
  SPB_CHECK_LAUNCH();
  *P = out;
  *S_out = S;
  return SP_OK;
}

int split_reduce(const double* P, int S, int64_t M, int64_t N, double alpha, double beta, double* C, int64_t ldc,
                 cudaStream_t s) {
  if (S > 8) {
    SPB_CUDA(launch_pdl((gemm_split_reduce_warp), dim3(ceil_div(M * N, 32)), dim3(256), 0, s, P, S, M, N, alpha, beta, C, ldc));
  } else {
    gemm_split_reduce<<<ceil_div(M * N, 256), 256, 0, s>>>(P, S, M, N, alpha, beta, C, ldc);
  }
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

}  // namespace spb
