// K1: deterministic sketch operator as an index gather (never materialises
// the n x n_c operator D / Omega).  Replaces apply_sketch for the stencil
// kinds (src/sketch.py:171-184) and gather_columns (src/sketch.py:201-211).
//
// Each thread owns one coarse column c and a strip of rows; the stencil
// table column (idx[:, c], w[:, c]) is loaded once into registers.  Loads of A
// are read-only (ld.global.nc) and issued 8 rows at a time so every thread has
// eight independent 8-byte requests in flight.  Adjacent coarse columns sit
// stride*8 bytes apart, so each warp touches the 32-byte sectors that hold
// grid points and nothing else: the algorithmic bytes of a gather.
#include "common.cuh"
#include "launch_count.cuh"

namespace spb {

template <typename TA>
__device__ __forceinline__ double load_nc(const TA* p) { return widen(__ldg(p)); }

constexpr int kGatherThreads = 128;
constexpr int kGatherRows = 8;     // rows per unrolled batch
constexpr int kMaxDepth = 16;      // stencil depth held in registers

// exact_copy=true: out = A[i, idx[c]] (gather_columns: keeps -0.0 and bits)
// exact_copy=false: out = sum_t fl(A * w) in t order starting from +0.0
template <typename TA, bool kExact>
__global__ void __launch_bounds__(kGatherThreads)
stencil_kernel(const TA* __restrict__ A, int64_t rows, int64_t lda,
               const int64_t* __restrict__ idx, const double* __restrict__ w,
               int depth, int64_t nc, int rows_per_cta, double* __restrict__ out,
               int64_t ldo) {
  const int64_t c = (int64_t)blockIdx.x * kGatherThreads + threadIdx.x;
  if (c >= nc) return;
  int64_t my_idx[kMaxDepth];
  double my_w[kMaxDepth];
#pragma unroll
  for (int t = 0; t < kMaxDepth; ++t) {
    if (t < depth) {
      my_idx[t] = idx[(int64_t)t * nc + c];
      my_w[t] = kExact ? 1.0 : w[(int64_t)t * nc + c];
    }
  }
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  for (int64_t i = r0; i < r1; i += kGatherRows) {
    double acc[kGatherRows];
    if (kExact) {
#pragma unroll
      for (int u = 0; u < kGatherRows; ++u)
        acc[u] = (i + u < r1) ? load_nc(A + (i + u) * lda + my_idx[0]) : 0.0;
    } else {
#pragma unroll
      for (int u = 0; u < kGatherRows; ++u) acc[u] = 0.0;
#pragma unroll
      for (int t = 0; t < kMaxDepth; ++t) {
        if (t >= depth) break;
        double v[kGatherRows];
#pragma unroll
        for (int u = 0; u < kGatherRows; ++u)
          v[u] = (i + u < r1) ? load_nc(A + (i + u) * lda + my_idx[t]) : 0.0;
#pragma unroll
        for (int u = 0; u < kGatherRows; ++u) acc[u] = __dadd_rn(acc[u], __dmul_rn(v[u], my_w[t]));
      }
    }
#pragma unroll
    for (int u = 0; u < kGatherRows; ++u)
      if (i + u < r1) out[(i + u) * ldo + c] = acc[u];
  }
}

// Deep stencils (global averaging with s > kMaxDepth): same arithmetic, table
// read from global per row batch.
template <typename TA>
__global__ void __launch_bounds__(kGatherThreads)
stencil_deep_kernel(const TA* __restrict__ A, int64_t rows, int64_t lda,
                    const int64_t* __restrict__ idx, const double* __restrict__ w,
                    int depth, int64_t nc, int rows_per_cta, double* __restrict__ out,
                    int64_t ldo) {
  const int64_t c = (int64_t)blockIdx.x * kGatherThreads + threadIdx.x;
  if (c >= nc) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  for (int64_t i = r0; i < r1; ++i) {
    double acc = 0.0;
    for (int t = 0; t < depth; ++t)
      acc = __dadd_rn(acc, __dmul_rn(load_nc(A + i * lda + idx[(int64_t)t * nc + c]),
                                     w[(int64_t)t * nc + c]));
    out[i * ldo + c] = acc;
  }
}

template <typename TA>
static int launch_stencil(const TA* A, int64_t rows, int64_t lda, const int64_t* idx,
                          const double* w, int depth, int64_t nc, bool exact, double* out,
                          int64_t ldo, cudaStream_t s) {
  const int gx = ceil_div(nc, kGatherThreads);
  // enough CTAs to cover ~4 waves of 148 SMs
  int gy = std::max(1, std::min<int>(ceil_div(rows, kGatherRows), (4 * kNumSMs * 8) / std::max(1, gx)));
  int rpc = ceil_div(rows, gy);
  rpc = ceil_div(rpc, kGatherRows) * kGatherRows;
  gy = ceil_div(rows, rpc);
  dim3 grid(gx, gy);
  if (exact) {
    stencil_kernel<TA, true><<<grid, kGatherThreads, 0, s>>>(A, rows, lda, idx, w, 1, nc, rpc, out, ldo);
  } else if (depth <= kMaxDepth) {
    stencil_kernel<TA, false><<<grid, kGatherThreads, 0, s>>>(A, rows, lda, idx, w, depth, nc, rpc, out, ldo);
  } else {
    stencil_deep_kernel<TA><<<grid, kGatherThreads, 0, s>>>(A, rows, lda, idx, w, depth, nc, rpc, out, ldo);
  }
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

int apply_stencil(const void* A, int a_dtype, int64_t rows, int64_t n, int64_t lda,
                  const int64_t* idx, const double* w, int depth, int64_t nc, bool exact,
                  double* out, int64_t ldo, cudaStream_t s) {
  SPB_REQUIRE(depth >= 1, "stencil depth must be >= 1");
  SPB_REQUIRE(!exact || depth == 1, "exact gather needs depth 1");
  SPB_REQUIRE(nc >= 1 && lda >= n && ldo >= nc, "bad stencil shapes");
  if (rows == 0) return SP_OK;
  if (a_dtype == SP_F64)
    return launch_stencil((const double*)A, rows, lda, idx, w, depth, nc, exact, out, ldo, s);
  if (a_dtype == SP_F32)
    return launch_stencil((const float*)A, rows, lda, idx, w, depth, nc, exact, out, ldo, s);
  set_error("unknown dtype tag");
  return SP_ECONFIG;
}

// ---------------------------------------------------- column validation ----
__global__ void check_columns_kernel(const int64_t* cols, int64_t count, int64_t n,
                                     unsigned int* seen, int* bad) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  int64_t c = cols[i];
  if (c < 0 || c >= n) {
    atomicOr(bad, 1);
    return;
  }
  unsigned int bit = 1u << (c & 31);
  unsigned int old = atomicOr(&seen[c >> 5], bit);
  if (old & bit) atomicOr(bad, 2);
}

int check_columns(const int64_t* cols, int64_t count, int64_t n, cudaStream_t s) {
  SPB_REQUIRE(count > 0, "empty column index set");
  Arena ar(s);
  const int64_t words = (n + 31) / 32;
  SPB_ALLOC(ar, unsigned int, seen, words + 1);
  int* bad = (int*)(seen + words);
  SPB_CUDA(cudaMemsetAsync(seen, 0, (words + 1) * sizeof(unsigned int), s));
  check_columns_kernel<<<ceil_div(count, 256), 256, 0, s>>>(cols, count, n, seen, bad);
  count_launch();
  SPB_CHECK_LAUNCH();
  int hbad = 0;
  SPB_TRY(read_small(&hbad, bad, sizeof(int), s));
  if (hbad & 1) {
    set_error("column index out of range [0, " + std::to_string(n) + ")");
    return SP_ECONFIG;
  }
  if (hbad & 2) {
    set_error("column indices must be distinct");
    return SP_ECONFIG;
  }
  return SP_OK;
}

}  // namespace spb
