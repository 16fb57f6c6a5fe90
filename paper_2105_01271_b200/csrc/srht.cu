// Range-finder test block Y = X Omega for the sketch-side subspace iteration
// (svd_top, pipeline.cu) as a subsampled randomized Hadamard transform:
//   Omega = D H S  (D random signs, H the Walsh-Hadamard matrix of the
//   zero-padded width 2^L, S b stratified column samples),
// i.e. each row of X is sign-flipped, Hadamard-transformed and sampled.
// A structured random embedding (Halko, Martinsson & Tropp 2011, sec. 4.6)
// in place of the dense Gaussian block: L 2^L additions per row instead of
// 2 b 2^L FMAs on the DMMA pipe, one read of X, no Omega in memory.  The
// block only has to capture the dominant column space; the Rayleigh-Ritz
// step and the convergence tests that follow are unchanged.
//
// One CTA per row (16..1024 threads, 16 elements each, widths up to 16384):
// the top 4 index bits are transformed in registers straight from the
// coalesced load, the rest in rounds of 4 bits through padded shared memory
// (a thread's 16 slots re-mapped to the round's bits), then the b sampled
// outputs are read out.  Non-finite input raises *flag (the
// reference checks the sketch before its QR, src/kernels.py:47-49).
// Fixed operation order: bitwise reproducible.
#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

__device__ __forceinline__ uint64_t srht_hash(uint64_t seed, uint64_t t) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ull + t * 0xD1B54A32D192ED03ull + 0x2545F4914F6CDD1Dull;
  z = (z ^ (z >> 31)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 29)) * 0x94D049BB133111EBull;
  return z ^ (z >> 32);
}

// stratified sample c in [0, b): one position in each of the b blocks of N / b
__device__ __forceinline__ int srht_sample(uint64_t seed, int c, int blk) {
  const uint64_t z = srht_hash(seed ^ 0x5851F42D4C957F2Dull, (uint64_t)c);
  return c * blk + (int)(z % (uint64_t)blk);
}

__device__ __forceinline__ int srht_pad(int j) { return j + (j >> 4); }

// element index of slot e of thread t in a round over bits [lo, lo + nb):
// bits [lo, lo+nb) = e's low nb bits, the thread index fills [0, lo) and
// [lo+nb, LT+nb), e's remaining 4 - nb bits go on top.
template <int LT>
__device__ __forceinline__ int srht_index(int t, int e, int lo, int nb) {
  const int el = e & ((1 << nb) - 1), eh = e >> nb;
  return (t & ((1 << lo) - 1)) | (el << lo) | ((t >> lo) << (lo + nb)) | (eh << (LT + nb));
}

// 16 elements per thread; butterflies over slot bits [0, nb)
__device__ __forceinline__ void srht_stages(double (&v)[16], int nb) {
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (s < nb) {
      const int h = 1 << s;
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if ((e & h) == 0) {
          const double a = v[e], c = v[e + h];
          v[e] = a + c;
          v[e + h] = a - c;
        }
    }
  }
}

// One CTA (2^LT threads) per row, N = 16 * 2^LT (zero-padded) elements:
// the coalesced load is the round over the top 4 bits; then rounds of 4
// bits through padded shared memory (the last one narrower if LT % 4 != 0).
// The transform of one row held as v[e] = element t + T e (sign applied
// here); writes the b sampled outputs to yrow.  Uniform barriers only.
template <int LT>
__device__ __forceinline__ void srht_row(double (&v)[16], uint64_t sg, int b, uint64_t seed, double* sr_smem,
                                         double* __restrict__ yrow, int* __restrict__ flag) {
  constexpr int T = 1 << LT, N = 16 * T;
  const int t = threadIdx.x;
  bool bad = false;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const double x = v[e];
    bad |= !isfinite(x);
    v[e] = __longlong_as_double(__double_as_longlong(x) ^ (long long)(((sg >> e) & 1ull) << 63));
  }
  if (__syncthreads_or(bad)) {
    if (t == 0 && flag) atomicOr(flag, 1);
  }
  srht_stages(v, 4);  // index bits [LT, LT + 4)
  int plo = LT, pnb = 4;  // layout of the values held
#pragma unroll
  for (int lo = 0; lo < LT; lo += 4) {
    const int nb = LT - lo < 4 ? LT - lo : 4;
#pragma unroll
    for (int e = 0; e < 16; ++e) sr_smem[srht_pad(srht_index<LT>(t, e, plo, pnb))] = v[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = sr_smem[srht_pad(srht_index<LT>(t, e, lo, nb))];
    __syncthreads();
    srht_stages(v, nb);
    plo = lo;
    pnb = nb;
  }
#pragma unroll
  for (int e = 0; e < 16; ++e) sr_smem[srht_pad(srht_index<LT>(t, e, plo, pnb))] = v[e];
  __syncthreads();
  for (int c = t; c < b; c += T) yrow[c] = sr_smem[srht_pad(srht_sample(seed, c, N / b))];
  __syncthreads();  // sr_smem is reused by the next row
}

// GATHER: the rows of X are gathered on the fly from A (X[row][j] =
// A[row][gidx[j]], exact copies, written to X as well): the coarse-column
// block C = A(:, I) and its test block Y come out of one pass over A (K1 fused
// with the range finder's first product).  RPC rows per CTA (the kernel is
// templated on it); one row per CTA is used: 2 rows held 75 -> 103
// registers, i.e. 3 -> 2 resident CTAs per SM, and the extra CTAs overlap one
// row's gather loads with another's transform better than the wider batch
// (measured: cfg2 rows 67.9 -> 60.3 us, cfg4-width rows 458 -> 386 us per
// 2000 rows).  Both modes give bit-identical Y.
template <int LT, bool GATHER, int RPC, typename TA>
__global__ void __launch_bounds__(1 << LT)
srht_kernel(int64_t rows, int64_t cols, const double* __restrict__ X, int64_t ldx, int b, uint64_t seed,
            double* __restrict__ Y, int64_t ldy, int* __restrict__ flag, const TA* __restrict__ A, int64_t lda,
            const int64_t* __restrict__ gidx, double* __restrict__ Xout, int64_t ychunk) {
  SPB_PDL_ENTRY();
  constexpr int T = 1 << LT;
  extern __shared__ double sr_smem[];  // srht_pad(N) doubles
  const int t = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.x * RPC;
  // chunk (blockIdx.y) of a row wider than the transform (gather mode): its
  // own random signs, the same Hadamard samples; partial Y at Y + chunk * ychunk
  const int chunk = blockIdx.y;
  const int64_t cbase = (int64_t)chunk * (16 * T);
  Y += chunk * ychunk;
  const uint64_t sg = srht_hash(chunk ? seed ^ (0xA24BAED4963EE407ull * (uint64_t)chunk) : seed,
                                (uint64_t)t);  // sign of element t + T e: bit e
  double v[RPC][16];
  if (GATHER) {
    int64_t gi[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int64_t j = cbase + t + (int64_t)T * e;
      gi[e] = j < cols ? __ldg(gidx + j) : 0;
    }
#pragma unroll
    for (int r = 0; r < RPC; ++r) {
      const bool live = row0 + r < rows;
      const TA* ar = A + (live ? row0 + r : 0) * lda;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int64_t j = cbase + t + (int64_t)T * e;
        v[r][e] = (live && j < cols) ? widen(__ldg(ar + gi[e])) : 0.0;
      }
    }
#pragma unroll
    for (int r = 0; r < RPC; ++r) {
      if (row0 + r >= rows) break;
      double* orow = Xout + (row0 + r) * ldx;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int64_t j = cbase + t + (int64_t)T * e;
        if (j < cols) orow[j] = v[r][e];
      }
    }
  } else {
#pragma unroll
    for (int r = 0; r < RPC; ++r) {
      const bool live = row0 + r < rows;
      const double* xr = X + (live ? row0 + r : 0) * ldx;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int64_t j = (int64_t)t + (int64_t)T * e;
        v[r][e] = (live && j < cols) ? xr[j] : 0.0;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RPC; ++r) {
    if (row0 + r >= rows) break;  // uniform
    srht_row<LT>(v[r], sg, b, seed, sr_smem, Y + (row0 + r) * ldy, flag);
  }
}

// padded width N = 16 * 2^LT = the next power of two >= cols (>= 256): a
// wider pad would leave the sampled Hadamard columns distinguished by their
// low bits only on the first `cols` rows (colliding samples)
static int srht_lt(int64_t cols) {
  int lt = 4;
  while (lt < 10 && ((int64_t)16 << lt) < cols) ++lt;
  return lt;
}

bool srht_ok(int64_t rows, int64_t cols, int b) {
  const int64_t n2 = (int64_t)16 << srht_lt(cols);
  return cols >= 1 && cols <= n2 && b >= 1 && b <= 32 && n2 % b == 0 && rows >= 1 && rows <= 0x7fffffff;
}

// gather mode: rows wider than the widest transform (16384) are cut into
// 16384-column chunks, each transformed with its own signs and the same
// samples; the partial test blocks are summed in chunk order (a block SRHT,
// Balabanov, Beaupere, Grigori & Lederer 2022: the columns of Omega stay
// orthogonal, Omega^T Omega = chunks * N * I)
constexpr int64_t kSrhtChunk = 16384;

bool srht_gather_ok(int64_t rows, int64_t cols, int b) {
  if (cols <= kSrhtChunk) return srht_ok(rows, cols, b);
  return b >= 1 && b <= 32 && kSrhtChunk % b == 0 && rows >= 1 && rows <= 0x7fffffff && cols / kSrhtChunk < 65535;
}

template <bool GATHER, typename TA>
static int srht_launch(int64_t rows, int64_t cols, const double* X, int64_t ldx, int b, uint64_t seed, double* Y,
                       int64_t ldy, int* flag, const TA* A, int64_t lda, const int64_t* gidx, double* Xout,
                       cudaStream_t s) {
  constexpr int RPC = 1;
  const int nchunk = (GATHER && cols > kSrhtChunk) ? (int)ceil_div(cols, kSrhtChunk) : 1;
  Arena ar(s);
  double* Yk = Y;
  int64_t ldyk = ldy, ychunk = 0;
  if (nchunk > 1) {
    Yk = ar.alloc<double>((size_t)nchunk * rows * b);
    if (!Yk) {
      set_error("srht chunk workspace allocation failed");
      return SP_ECUDA;
    }
    ldyk = b;
    ychunk = rows * b;
  }
  const int lt = srht_lt(cols);
  const int64_t n2 = (int64_t)16 << lt;
  const size_t smem = (size_t)(n2 + n2 / 16) * sizeof(double);
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    SPB_CUDA(cudaFuncSetAttribute(srht_kernel<9, GATHER, RPC, TA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    SPB_CUDA(cudaFuncSetAttribute(srht_kernel<10, GATHER, RPC, TA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_dev = dev;
  }
  const dim3 grid((unsigned)((rows + RPC - 1) / RPC), (unsigned)nchunk);
  switch (lt) {
#define SPB_SRHT_LT(L)                                                                                              \
  case L:                                                                                                           \
    SPB_CUDA(launch_pdl((srht_kernel<L, GATHER, RPC, TA>), grid, dim3(1 << L), smem, s, rows, cols, X, ldx, b, seed, \
                        Yk, ldyk, flag, A, lda, gidx, Xout, ychunk));                                               \
    break;
    SPB_SRHT_LT(4) SPB_SRHT_LT(5) SPB_SRHT_LT(6) SPB_SRHT_LT(7) SPB_SRHT_LT(8) SPB_SRHT_LT(9) SPB_SRHT_LT(10)
#undef SPB_SRHT_LT
    default:
      set_error("srht: width out of range");
      return SP_ECONFIG;
  }
  count_launch();
  SPB_CHECK_LAUNCH();
  if (nchunk > 1) return split_reduce(Yk, nchunk, rows, b, 1.0, 0.0, Y, ldy, s);
  return SP_OK;
}

// Y (rows x b, ld ldy) = X D H S.  Returns SP_ECONFIG when the shape is out of
// the kernel's range (the caller falls back to a dense block on the GEMM).
int srht_sketch(int64_t rows, int64_t cols, const double* X, int64_t ldx, int b, uint64_t seed, double* Y,
                int64_t ldy, int* flag, cudaStream_t s) {
  if (!srht_ok(rows, cols, b)) {
    set_error("srht_sketch: shape out of range");
    return SP_ECONFIG;
  }
  return srht_launch<false, double>(rows, cols, X, ldx, b, seed, Y, ldy, flag, nullptr, 0, nullptr, nullptr, s);
}

// C (rows x cols, ld ldc) = A(:, gidx) (exact copies) and Y = C D H S, one pass.
int srht_gather(const void* A, int a_dtype, int64_t rows, int64_t lda, const int64_t* gidx, int64_t cols, double* C,
                int64_t ldc, int b, uint64_t seed, double* Y, int64_t ldy, int* flag, cudaStream_t s) {
  if (!srht_gather_ok(rows, cols, b)) {
    set_error("srht_gather: shape out of range");
    return SP_ECONFIG;
  }
  if (a_dtype == SP_F32)
    return srht_launch<true, float>(rows, cols, C, ldc, b, seed, Y, ldy, flag, (const float*)A, lda, gidx, C, s);
  return srht_launch<true, double>(rows, cols, C, ldc, b, seed, Y, ldy, flag, (const double*)A, lda, gidx, C, s);
}

}  // namespace spb
