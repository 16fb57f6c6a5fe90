// K2 (TMA version): Y (n x r) = A^T Z with the tiles of A streamed by the TMA
// bulk-copy engine into a 4-stage shared-memory ring.
//
// Persistent, one CTA per SM: CTA b owns the contiguous column slab
// [b*n/G, (b+1)*n/G) (rounded to 16-byte boundaries) and streams ALL m rows
// of it, so every CTA does the same amount of work, there is no split-K, no
// partial buffer and no reduction kernel -- A is read exactly once and Y is
// written once.  Warp 8 is the producer: one elected lane issues, per stage,
// 8 row-segment bulk copies of A (cp.async.bulk ... complete_tx) plus the
// matching 8 rows of Z on a full/empty mbarrier pair.  Warps 0-7 consume:
// each thread owns 16 bytes of columns (2 x f64 or 4 x f32) and keeps its
// V x R FP64 accumulator in registers; the Z row is a shared-memory broadcast.
// Bytes in flight per SM = 3 stages x 64 KB, independent of register pressure
// (16 rows per stage: fewer, larger stages measured 0.83 -> 0.90 of the HBM
// roofline at cfg2, where a CTA's row segment is only 3.5 KB).
#include <cstdlib>
#include <type_traits>

#include "async.cuh"
#include "common.cuh"
#include "launch_count.cuh"

namespace spb {

constexpr int kTmaConsumers = 256;
constexpr int kTmaThreads = kTmaConsumers + 32;
constexpr int kTmaRows = 16;      // rows per stage
constexpr int kTmaStages = 3;
constexpr int kTmaRowBytes = kTmaConsumers * 16;  // 4 KB of A per row per tile

// MMA variant: the products run on the FP64 tensor pipe (mma.sync m8n8k4,
// M = 8 columns of A, N = 8 columns of Z, K = 4 rows): one LDS.128 of A feeds
// V DMMAs (256 FMAs each) instead of V * R scalar DFMAs with R broadcast loads
// of Z -- ~6x fewer issued instructions per byte of A, which is what keeps the
// pass at the HBM roofline when a sustained run is power-capped (the scalar
// loop issues 14 TFLOP/s of DFMA at cfg4).  Rows are pitched 32 bytes past 4 KB
// so the fragment loads (4 rows x 8 lanes x 16 bytes per quarter warp) are
// bank-conflict free.
template <int R, bool MMA>
struct TmaLayout {
  static constexpr int kRowPitch = kTmaRowBytes + (MMA ? 32 : 0);
  static constexpr int kZStage = kTmaRows * R * 8;                       // bytes of Z per stage
  static constexpr int kZStagePad = (kZStage + 127) / 128 * 128;
  static constexpr int kZOff = (kTmaRows * kRowPitch + 127) / 128 * 128;
  static constexpr int kStageBytes = kZOff + kZStagePad;
  static constexpr int kSmem = kTmaStages * kStageBytes;
};

__device__ __forceinline__ void k2_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int R, typename TA, bool MMA>
__global__ void __launch_bounds__(kTmaThreads, 1)
skinny_tma_kernel(const TA* __restrict__ A, int64_t m, int64_t n, int64_t lda, const double* __restrict__ Zc,
                  double* __restrict__ Y, int64_t ldy, int splits) {
  SPB_PDL_ENTRY();
  constexpr int V = 16 / sizeof(TA);
  constexpr int TC = kTmaConsumers * V;  // columns per tile
  using L = TmaLayout<R, MMA>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kTmaStages];
  __shared__ __align__(8) uint64_t empty[kTmaStages];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // contiguous, 16-byte aligned column slab of this CTA; with splits > 1 the
  // rows are also divided (CTA b: row part b % splits of slab b / splits) and
  // each part writes its own partial Y (summed by skinny_split_reduce)
  const int64_t units = n / V;  // n % V == 0 is a launch precondition
  const int nslab = gridDim.x / splits, sl = blockIdx.x / splits, part = blockIdx.x % splits;
  const int64_t cb = (units * sl / nslab) * V;
  const int64_t ce = (units * (sl + 1) / nslab) * V;
  const int64_t rb = (m * part / splits) / kTmaRows * kTmaRows;
  const int64_t re = part + 1 == splits ? m : (m * (part + 1) / splits) / kTmaRows * kTmaRows;
  if (splits > 1) Y += (int64_t)part * n * ldy;

  if (tid == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumers / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == kTmaConsumers / 32) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int64_t c0 = cb; c0 < ce; c0 += TC) {
        const uint32_t seg = (uint32_t)(imin64(TC, ce - c0) * sizeof(TA));
        for (int64_t r0 = rb; r0 < re; r0 += kTmaRows) {
          const int nr = (int)imin64(kTmaRows, re - r0);
          unsigned char* sb = smem + stage * L::kStageBytes;
          mbar_wait(&empty[stage], ph ^ 1);
          const uint32_t zbytes = (uint32_t)(nr * R * 8);
          mbar_arrive_expect_tx(&full[stage], nr * seg + ((zbytes + 15) / 16) * 16);
          for (int i = 0; i < nr; ++i)
            bulk_g2s(sb + i * L::kRowPitch, A + (r0 + i) * lda + c0, seg, &full[stage]);
          bulk_g2s(sb + L::kZOff, Zc + r0 * R, ((zbytes + 15) / 16) * 16, &full[stage]);
          if (++stage == kTmaStages) {
            stage = 0;
            ph ^= 1;
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  int stage = 0;
  uint32_t ph = 0;
  if constexpr (MMA) {
    // warp w owns columns [w * 32 V, (w + 1) * 32 V) of the tile; lane (g, t):
    // fragment row t of each 4-row step, the V adjacent columns 4 V j + V g ..
    // of column group j (each a separate 8-column DMMA tile: m index g)
    constexpr int NT = (R + 7) / 8;  // 8-wide tiles of Z columns
    const int g = lane >> 2, t4 = lane & 3;
    for (int64_t c0 = cb; c0 < ce; c0 += TC) {
      double acc[4][V][NT][2];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int q = 0; q < NT; ++q) acc[j][v][q][0] = acc[j][v][q][1] = 0.0;
      for (int64_t r0 = rb; r0 < re; r0 += kTmaRows) {
        const int nr = (int)imin64(kTmaRows, re - r0);
        const unsigned char* sb = smem + stage * L::kStageBytes;
        const double* zs = reinterpret_cast<const double*>(sb + L::kZOff);
        mbar_wait(&full[stage], ph);
        // full stages take the unguarded body (no selects in the hot loop);
        // the last, ragged row block masks rows past it (stale bytes)
        auto body = [&](auto guard_tag) {
          constexpr bool kGuard = decltype(guard_tag)::value;
#pragma unroll
          for (int ks = 0; ks < kTmaRows / 4; ++ks) {
            const int row = 4 * ks + t4;
            const bool live = !kGuard || row < nr;
            double b[NT];
#pragma unroll
            for (int q = 0; q < NT; ++q) b[q] = (live && 8 * q + g < R) ? zs[row * R + 8 * q + g] : 0.0;
            const unsigned char* ap = sb + row * L::kRowPitch + (warp * 32 + g) * 16;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              double a[V];
              if constexpr (V == 2) {
                const double2 x = *reinterpret_cast<const double2*>(ap + j * 128);
                a[0] = x.x;
                a[1] = x.y;
              } else {
                const float4 x = *reinterpret_cast<const float4*>(ap + j * 128);
                a[0] = x.x;
                a[1] = x.y;
                a[2] = x.z;
                a[3] = x.w;
              }
#pragma unroll
              for (int v = 0; v < V; ++v) {
                const double av = live ? a[v] : 0.0;
#pragma unroll
                for (int q = 0; q < NT; ++q) k2_dmma(acc[j][v][q][0], acc[j][v][q][1], av, b[q]);
              }
            }
          }
        };
        if (nr == kTmaRows)
          body(std::false_type{});
        else
          body(std::true_type{});
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == kTmaStages) {
          stage = 0;
          ph ^= 1;
        }
      }
      // C fragment: row g (the column of A), columns 2 t4, 2 t4 + 1 of each Z tile
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int64_t col = c0 + (int64_t)(warp * 32 + j * 8 + g) * V + v;
          if (col < ce) {
#pragma unroll
            for (int q = 0; q < NT; ++q)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int c = 8 * q + 2 * t4 + e;
                if (c < R) Y[col * ldy + c] = acc[j][v][q][e];
              }
          }
        }
    }
    return;
  }
  for (int64_t c0 = cb; c0 < ce; c0 += TC) {
    const int64_t col = c0 + (int64_t)tid * V;
    double acc[V][R];
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int c = 0; c < R; ++c) acc[v][c] = 0.0;
    for (int64_t r0 = rb; r0 < re; r0 += kTmaRows) {
      const int nr = (int)imin64(kTmaRows, re - r0);
      const unsigned char* sb = smem + stage * L::kStageBytes;
      const double* zs = reinterpret_cast<const double*>(sb + L::kZOff);
      mbar_wait(&full[stage], ph);
      if (nr == kTmaRows) {
#pragma unroll
        for (int i = 0; i < kTmaRows; ++i) {
          double a[V];
          if constexpr (V == 2) {
            const double2 x = *reinterpret_cast<const double2*>(sb + i * L::kRowPitch + tid * 16);
            a[0] = x.x;
            a[1] = x.y;
          } else {
            const float4 x = *reinterpret_cast<const float4*>(sb + i * L::kRowPitch + tid * 16);
            a[0] = x.x;
            a[1] = x.y;
            a[2] = x.z;
            a[3] = x.w;
          }
#pragma unroll
          for (int c = 0; c < R; ++c) {
            const double z = zs[i * R + c];
#pragma unroll
            for (int v = 0; v < V; ++v) acc[v][c] = fma(a[v], z, acc[v][c]);
          }
        }
      } else {
        for (int i = 0; i < nr; ++i) {
          const TA* ap = reinterpret_cast<const TA*>(sb + i * L::kRowPitch) + tid * V;
#pragma unroll
          for (int c = 0; c < R; ++c) {
            const double z = zs[i * R + c];
#pragma unroll
            for (int v = 0; v < V; ++v) acc[v][c] = fma((double)ap[v], z, acc[v][c]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kTmaStages) {
        stage = 0;
        ph ^= 1;
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if (col + v < ce) {
#pragma unroll
        for (int c = 0; c < R; ++c) Y[(col + v) * ldy + c] = acc[v][c];
      }
    }
  }
}

// Y = sum_p Ypart[p] (fixed order)
__global__ void skinny_split_reduce(int splits, int64_t count, const double* __restrict__ part,
                                    double* __restrict__ Y) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  double a = part[e];
  for (int p = 1; p < splits; ++p) a += part[(int64_t)p * count + e];
  Y[e] = a;
}

template <int R, typename TA, bool MMA>
static int skinny_tma_launch_v(const TA* A, int64_t m, int64_t n, int64_t lda, const double* Zc, double* Y,
                               int64_t ldy, cudaStream_t s) {
  using L = TmaLayout<R, MMA>;
  constexpr int V = 16 / sizeof(TA);
  static int attr_dev = -1;  // set once per device (host overhead sits on the critical path)
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    SPB_CUDA(cudaFuncSetAttribute(skinny_tma_kernel<R, TA, MMA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  L::kSmem));
    attr_dev = dev;
  }
  const int64_t units = n / V;
  // Row splitting (CTA = row part x column slab, partial Y + one reduction)
  // lengthens each CTA's row segments; measured slower than full-height slabs
  // at cfg2 (209 / 219 us for 2 / 4 parts vs 191 us), so it is off unless
  // SPB_K2_SPLIT asks for it (experiments only).
  static const int env_splits = [] {
    const char* e = getenv("SPB_K2_SPLIT");
    return e ? std::max(1, std::min(8, atoi(e))) : 1;
  }();
  int splits = env_splits;
  if (ldy != R || m < (int64_t)2 * kTmaRows * splits) splits = 1;
  while (splits > 1 && units / 16 < (kNumSMs / splits)) --splits;
  int grid = (int)std::min<int64_t>(kNumSMs / splits, std::max<int64_t>(1, units / 16)) * splits;
  Arena ar(s);
  double* out = Y;
  if (splits > 1) {
    out = ar.alloc<double>((size_t)splits * n * R);
    if (!out) {
      set_error("skinny split workspace allocation failed");
      return SP_ECUDA;
    }
  }
  SPB_CUDA(launch_pdl((skinny_tma_kernel<R, TA, MMA>), dim3(grid), dim3(kTmaThreads), L::kSmem, s, A, m, n, lda, Zc, out, splits > 1 ? R : ldy, splits));
  count_launch();
  SPB_CHECK_LAUNCH();
  if (splits > 1) {
    skinny_split_reduce<<<ceil_div(n * R, 256), 256, 0, s>>>(splits, n * R, out, Y);
    count_launch();
    SPB_CHECK_LAUNCH();
  }
  return SP_OK;
}

template <int R, typename TA>
int skinny_tma_launch(const TA* A, int64_t m, int64_t n, int64_t lda, const double* Zc, double* Y, int64_t ldy,
                      cudaStream_t s) {
  // SPB_K2_FMA=1: the scalar-DFMA consumers (experiments / comparison)
  static const bool fma_loop = getenv("SPB_K2_FMA") != nullptr;
  if (fma_loop) return skinny_tma_launch_v<R, TA, false>(A, m, n, lda, Zc, Y, ldy, s);
  return skinny_tma_launch_v<R, TA, true>(A, m, n, lda, Zc, Y, ldy, s);
}

// Preconditions of the bulk-copy path: 16-byte aligned base, row pitch and
// slab boundaries (n a multiple of the 16-byte vector).
bool skinny_tma_ok(const void* A, int a_dtype, int64_t n, int64_t lda) {
  const int es = a_dtype == SP_F64 ? 8 : 4;
  const int V = 16 / es;
  return (reinterpret_cast<uintptr_t>(A) % 16 == 0) && ((lda * es) % 16 == 0) && (n % V == 0) && n >= V;
}

#define SPB_INST(RR)                                                                                       \
  template int skinny_tma_launch<RR, double>(const double*, int64_t, int64_t, int64_t, const double*, double*, \
                                             int64_t, cudaStream_t);                                        \
  template int skinny_tma_launch<RR, float>(const float*, int64_t, int64_t, int64_t, const double*, double*,   \
                                            int64_t, cudaStream_t);
SPB_INST(1) SPB_INST(2) SPB_INST(3) SPB_INST(4) SPB_INST(5) SPB_INST(6) SPB_INST(7) SPB_INST(8)
SPB_INST(9) SPB_INST(10) SPB_INST(11) SPB_INST(12) SPB_INST(13) SPB_INST(14) SPB_INST(15) SPB_INST(16)
#undef SPB_INST

}  // namespace spb
