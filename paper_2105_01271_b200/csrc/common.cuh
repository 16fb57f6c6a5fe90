// Shared helpers for the sketchpress-b200 device library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <algorithm>

#include "../../include/sketchpress_b200.h"

namespace spb {

// ---------------------------------------------------------------- errors ----
// The C-ABI returns an int status (SP_OK / SP_ECONFIG / SP_EIO / SP_ENUMERICAL /
// SP_ECUDA) and keeps a thread-local message for sp_last_error().
void set_error(const std::string& msg);
const char* last_error();

struct Status {
  int code = SP_OK;
  int warn = 0;
};

#define SPB_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess) {                                                  \
      cudaGetLastError(); /* clear it: a failed call must not poison the next */ \
      ::spb::set_error(std::string(#call) + ": " + cudaGetErrorString(_e));    \
      return SP_ECUDA;                                                        \
    }                                                                         \
  } while (0)

#define SPB_CHECK_LAUNCH()                                                    \
  do {                                                                        \
    cudaError_t _e = cudaGetLastError();                                      \
    if (_e != cudaSuccess) {                                                  \
      ::spb::set_error(std::string("kernel launch (") + __FILE__ + ":" + std::to_string(__LINE__) + "): " + \
                       cudaGetErrorString(_e));                               \
      return SP_ECUDA;                                                        \
    }                                                                         \
  } while (0)

#define SPB_TRY(expr)                                                         \
  do {                                                                        \
    int _s = (expr);                                                          \
    if (_s != SP_OK) return _s;                                               \
  } while (0)

#define SPB_REQUIRE(cond, msg)                                                \
  do {                                                                        \
    if (!(cond)) {                                                            \
      ::spb::set_error(msg);                                                  \
      return SP_ECONFIG;                                                      \
    }                                                                         \
  } while (0)

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

constexpr int kNumSMs = 148;

// ------------------------------------------------------- device helpers ----
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T>
__device__ __forceinline__ double widen(T x) { return (double)x; }

// FP64 reciprocal / reciprocal square root from the MUFU approximations
// (rcp / rsqrt .approx.ftz.f64) refined by two Newton steps: ~1 ulp, at a
// fraction of the latency of the IEEE-rounded forms on the serial chains of
// the Householder and Jacobi steps.  The argument must be normal and finite
// (and > 0 for the rsqrt); callers guard the range.
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y * y, 1.0);
  y = fma(0.5 * y, e, y);
  e = fma(-x, y * y, 1.0);
  return fma(0.5 * y, e, y);
}
__device__ __forceinline__ bool fast_range(double x) { return x > 1e-290 && x < 1e290; }

// Staging global -> shared without a register round trip: every thread
// issues all of its 8-byte copies back to back (zero-fill when !pred; gmem
// must still be a mapped address then, e.g. the array base), so a staging
// loop costs one memory latency instead of one per iteration.
__device__ __forceinline__ void cp_async_f64(double* smem, const double* gmem, bool pred) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem), "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Counter-based hash -> uniform double in (-1, 1); used for the random test
// blocks of the range finder (any full-rank block works; no parity with numpy).
__device__ __forceinline__ double hash_uniform(uint64_t seed, uint64_t i) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ull + i * 0xD1B54A32D192ED03ull + 0x8CB92BA72F3D8DD7ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return ((double)(z >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

// Host-side trace of the pipelines' critical path (SPB_HOST_TRACE=1):
// host_mark(tag) records (tag, steady-clock us); sp_host_trace() dumps them.
void host_mark(const char* tag);

// Diagnostic phase timers (build with SPB_NVCC_EXTRA=-DSPB_PHASE_TRACE):
// SPB_TMARK(i) records clock64() into slot i, SPB_TPRINT(name, n) prints the
// n - 1 phase durations from the calling thread.
#ifdef SPB_PHASE_TRACE
#define SPB_TDECL long long spb_tm[12] = {0}
#define SPB_TMARK(i) spb_tm[i] = clock64()
#define SPB_TPRINT(name, n)                                                            \
  do {                                                                                 \
    printf("%s:", name);                                                               \
    for (int _i = 1; _i < (n); ++_i) printf(" %lld", spb_tm[_i] - spb_tm[_i - 1]);     \
    printf(" cyc\n");                                                                  \
  } while (0)
#else
#define SPB_TDECL
#define SPB_TMARK(i)
#define SPB_TPRINT(name, n)
#endif

// ------------------------------------------- programmatic dependent launch ----
// The pipelines are chains of small dependent kernels on one stream; with
// programmatic stream serialization a kernel is scheduled while its
// predecessor drains instead of after it completes.  Every kernel launched
// with launch_pdl starts with SPB_PDL_ENTRY(): it lets its own successor
// launch, then waits (griddepcontrol.wait) until the predecessor grid has
// completed and its memory is visible -- so no kernel touches global memory
// before its inputs are final.  Both instructions are no-ops for a kernel
// launched without the attribute.
#define SPB_PDL_ENTRY()                                              \
  do {                                                               \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    asm volatile("griddepcontrol.wait;" ::: "memory");              \
  } while (0)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ------------------------------------------------------ workspace arena ----
// Stream-ordered scratch.  The pipelines allocate a few dozen small
// workspaces per call; cudaMallocAsync + cudaFreeAsync cost ~2-4 us of host
// time each, which sits on the critical path right after every host
// synchronisation.  ws_alloc / ws_free keep freed blocks in per-(device,
// stream) free lists keyed by rounded size (reuse is stream ordered on the
// same stream, hence safe); overflow past the cache cap (64 GB per device)
// goes straight back to the CUDA mempool (cudaFreeAsync).  On an
// allocation failure the cache is drained (device synchronised) and the
// allocation retried once.
void* ws_alloc(size_t bytes, cudaStream_t s);
void ws_free(void* p, size_t bytes, cudaStream_t s);
void ws_release_all();  // drop every cached block (synchronises the device)

class Arena {
 public:
  explicit Arena(cudaStream_t s) : stream_(s) {}
  ~Arena() {
    for (int i = n_ - 1; i >= 0; --i) ws_free(ptrs_[i], sizes_[i], stream_);
  }
  template <typename T>
  T* alloc(size_t count) {
    if (count == 0) count = 1;
    void* p = nullptr;
    if (n_ >= kMax || (p = ws_alloc(count * sizeof(T), stream_)) == nullptr) {
      failed_ = true;
      return nullptr;
    }
    sizes_[n_] = count * sizeof(T);
    ptrs_[n_++] = p;
    return static_cast<T*>(p);
  }
  bool failed() const { return failed_; }
  cudaStream_t stream() const { return stream_; }

 private:
  static constexpr int kMax = 256;
  cudaStream_t stream_;
  void* ptrs_[kMax];
  size_t sizes_[kMax];
  int n_ = 0;
  bool failed_ = false;
};

// Small device -> host reads through a per-thread pinned staging buffer:
// pageable cudaMemcpyAsync is staged by the driver and blocks the host thread
// per copy; pinned copies are queued and complete at one stream sync.
//   PinnedReads rd(s); rd.add(&h, dptr, 4); ...; SPB_TRY(rd.sync());
class PinnedReads {
 public:
  explicit PinnedReads(cudaStream_t s) : s_(s) {}
  int add(void* host_dst, const void* dev_src, size_t bytes);
  int sync();  // cudaStreamSynchronize + scatter into the destinations

 private:
  static constexpr int kMax = 8;
  cudaStream_t s_;
  void* dst_[kMax];
  size_t off_[kMax], len_[kMax];
  size_t used_ = 0;
  int n_ = 0;
};

// one small device -> host read, then a stream sync
int read_small(void* host_dst, const void* dev_src, size_t bytes, cudaStream_t s);

#define SPB_ALLOC(arena, T, var, count)                                       \
  T* var = (arena).template alloc<T>(count);                                  \
  if (!var) {                                                                 \
    ::spb::set_error("device workspace allocation failed: " #var);            \
    return SP_ECUDA;                                                          \
  }

}  // namespace spb
