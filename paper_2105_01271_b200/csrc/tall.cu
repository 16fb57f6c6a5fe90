// Tall-skinny products of the sketch-sized algebra, where the 64x64 DMMA
// tiles of K3 waste most of their work (widths <= 64, rows up to n):
//   tall_gram : G = alpha X^T Y + beta G   (X: rows x c, Y: rows x d)
//   tall_mul  : O = alpha X M + beta O     (X: rows x c, M: c x d)
// Both stage row tiles of the tall operand in shared memory with coalesced
// loads (one pass over it) and are latency-, not FLOP-, bound at the path's
// shapes (65536 x 7, 4096 x 32).  tall_gram reduces per-CTA partials in a
// fixed order (bitwise reproducible).
#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

constexpr int kTallMax = 64;
constexpr int kTgThreads = 256;
constexpr int kTgTile = 64;  // rows per staged tile

__device__ __forceinline__ int round_up_dev(int x, int m) { return (x + m - 1) / m * m; }

// Copies rows [base, base + nr) of X (cols c) into s (stride sp, zero pad up
// to sp - 1 columns and up to `tile` rows).  Four threads per row (no integer
// division in the address computation; each row's bytes are read by
// neighbouring lanes).
__device__ __forceinline__ void stage_rows(double* s, int sp, int tile, const double* X, int64_t ldx,
                                           int64_t base, int nr, int c) {
  const int width = sp - 1;
  for (int rr = threadIdx.x >> 2; rr < tile; rr += blockDim.x >> 2) {
    const double* src = X + (base + (rr < nr ? rr : 0)) * ldx;
    for (int cc = threadIdx.x & 3; cc < width; cc += 4) {
      const bool ok = rr < nr && cc < c;
      cp_async_f64(&s[rr * sp + cc], ok ? src + cc : X, ok);
    }
  }
}

// partial[blk] = X_blk^T Y_blk over the CTA's rows.  Thread t owns an MT x MT
// output micro-tile (t % nmicro) and the rows rr = t / nmicro (mod G) of each
// staged tile; the G row-group partials are summed in a fixed order at the end.
template <int MT>
__global__ void __launch_bounds__(kTgThreads)
tall_gram_kernel(int64_t rows, int c, const double* __restrict__ X, int64_t ldx, int d,
                 const double* __restrict__ Y, int64_t ldy, int64_t rows_per_cta, double* __restrict__ partial) {
  extern __shared__ double tg_smem[];
  const int cp = round_up_dev(c, MT) + 1, dp = round_up_dev(d, MT) + 1;
  const int stage = kTgTile * (cp + dp);  // doubles per pipeline stage
  const int nmc = (c + MT - 1) / MT, nmd = (d + MT - 1) / MT, nmicro = nmc * nmd;
  const int G = kTgThreads / nmicro;
  const int mt = threadIdx.x % nmicro, rg = threadIdx.x / nmicro;
  const bool active = rg < G;
  const int i0 = (mt / nmd) * MT, j0 = (mt % nmd) * MT;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = imin64(rows, r0 + rows_per_cta);
  const int ntile = (int)((r1 - r0 + kTgTile - 1) / kTgTile);
  double acc[MT][MT];
#pragma unroll
  for (int u = 0; u < MT; ++u)
#pragma unroll
    for (int v = 0; v < MT; ++v) acc[u][v] = 0.0;
  auto issue = [&](int t) {
    const int64_t base = r0 + (int64_t)t * kTgTile;
    const int nr = (int)imin64(kTgTile, r1 - base);
    double* xs = tg_smem + (t & 1) * stage;
    stage_rows(xs, cp, kTgTile, X, ldx, base, nr, c);
    stage_rows(xs + kTgTile * cp, dp, kTgTile, Y, ldy, base, nr, d);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // two-stage cp.async pipeline over the CTA's row tiles
  if (ntile > 0) issue(0);
  for (int t = 0; t < ntile; ++t) {
    if (t + 1 < ntile) {
      issue(t + 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* xs = tg_smem + (t & 1) * stage;
    const double* ys = xs + kTgTile * cp;
    const int nr = (int)imin64(kTgTile, r1 - (r0 + (int64_t)t * kTgTile));
    if (active) {
      for (int rr = rg; rr < nr; rr += G) {
        double xv[MT], yv[MT];
#pragma unroll
        for (int u = 0; u < MT; ++u) {
          xv[u] = xs[rr * cp + i0 + u];
          yv[u] = ys[rr * dp + j0 + u];
        }
#pragma unroll
        for (int u = 0; u < MT; ++u)
#pragma unroll
          for (int v = 0; v < MT; ++v) acc[u][v] = fma(xv[u], yv[v], acc[u][v]);
      }
    }
    __syncthreads();  // stage (t & 1) is refilled by issue(t + 2)
  }
  // row-group partials -> shared (reusing the tiles), fixed-order sum
  double* red = tg_smem;  // [G][nmicro][MT*MT]
  if (active) {
#pragma unroll
    for (int u = 0; u < MT; ++u)
#pragma unroll
      for (int v = 0; v < MT; ++v) red[(rg * nmicro + mt) * MT * MT + u * MT + v] = acc[u][v];
  }
  __syncthreads();
  const int nout = c * d;
  for (int o = threadIdx.x; o < nout; o += kTgThreads) {
    const int i = o / d, j = o - (o / d) * d;
    const int m = (i / MT) * nmd + j / MT, uv = (i % MT) * MT + (j % MT);
    double t = 0.0;
    for (int g = 0; g < G; ++g) t += red[(g * nmicro + m) * MT * MT + uv];
    partial[(int64_t)blockIdx.x * nout + o] = t;
  }
}

template <int MT>
static int launch_tall_gram(int nb, int64_t rows, int c, const double* X, int64_t ldx, int d, const double* Y,
                            int64_t ldy, int64_t rpc, double* part, cudaStream_t s) {
  const int cp = (c + MT - 1) / MT * MT + 1, dp = (d + MT - 1) / MT * MT + 1;
  const size_t tile = (size_t)2 * kTgTile * (cp + dp), red = (size_t)kTgThreads * MT * MT;
  const size_t smem = (tile > red ? tile : red) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    SPB_CUDA(cudaFuncSetAttribute(tall_gram_kernel<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    attr = true;
  }
  tall_gram_kernel<MT><<<nb, kTgThreads, smem, s>>>(rows, c, X, ldx, d, Y, ldy, rpc, part);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

// per-CTA partials only (nb_max slabs of c x d available in part; *nb_out = used)
int tall_gram_partials(int64_t rows, int c, const double* X, int64_t ldx, int d, const double* Y, int64_t ldy,
                       double* part, int nb_max, int* nb_out, cudaStream_t s) {
  SPB_REQUIRE(c >= 1 && d >= 1 && c <= kTallMax && d <= kTallMax, "tall_gram supports widths <= 64");
  SPB_REQUIRE(rows >= 1 && nb_max >= 1, "tall_gram needs rows >= 1");
  int nb = (int)std::min<int64_t>(nb_max, ceil_div(rows, 2 * kTgTile));
  const int64_t rpc = ceil_div(ceil_div(rows, nb), kTgTile) * (int64_t)kTgTile;
  nb = (int)ceil_div(rows, rpc);
  *nb_out = nb;
  return (c <= 32 && d <= 32) ? launch_tall_gram<2>(nb, rows, c, X, ldx, d, Y, ldy, rpc, part, s)
                              : launch_tall_gram<4>(nb, rows, c, X, ldx, d, Y, ldy, rpc, part, s);
}

int tall_gram(int64_t rows, int c, const double* X, int64_t ldx, int d, const double* Y, int64_t ldy,
              double alpha, double beta, double* G, int64_t ldg, cudaStream_t s) {
  SPB_REQUIRE(c >= 1 && d >= 1 && c <= kTallMax && d <= kTallMax, "tall_gram supports widths <= 64");
  SPB_REQUIRE(rows >= 1, "tall_gram needs rows >= 1");
  int nb = (int)std::min<int64_t>(4 * kNumSMs, ceil_div(rows, 2 * kTgTile));
  const int64_t rpc = ceil_div(ceil_div(rows, nb), kTgTile) * (int64_t)kTgTile;
  nb = (int)ceil_div(rows, rpc);
  Arena ar(s);
  SPB_ALLOC(ar, double, part, (size_t)nb * c * d);
  const int st = (c <= 32 && d <= 32)
                     ? launch_tall_gram<2>(nb, rows, c, X, ldx, d, Y, ldy, rpc, part, s)
                     : launch_tall_gram<4>(nb, rows, c, X, ldx, d, Y, ldy, rpc, part, s);
  if (st != SP_OK) return st;
  return split_reduce(part, nb, c, d, alpha, beta, G, ldg, s);
}

// O = alpha X M + beta O.  Row tiles of R = min(512, 2048 / d) rows are
// visited grid-stride (M staged once per CTA); within a tile each thread forms
// output elements t, t + 256, ... of the row-major R x d block (coalesced
// loads and stores whatever d is; the (row, column) of the next element is
// stepped without division).  Each output row depends only on the same row
// of X, and a tile is staged before any of it is written, so O may alias X
// (same rows, any columns).
constexpr int kTmThreads = 256;

__global__ void __launch_bounds__(kTmThreads)
tall_mul_kernel(int64_t rows, int c, const double* X, int64_t ldx, int d, const double* __restrict__ M,
                int64_t ldm, double alpha, double beta, double* O, int64_t ldo, const double* __restrict__ top,
                int64_t ldt, int64_t top_rows, int rpc) {
  SPB_PDL_ENTRY();
  extern __shared__ __align__(16) double tm_smem[];
  const int sp = c + 1;
  double* ms = tm_smem;          // [c][d]
  double* ts = tm_smem + c * d;  // [rpc][sp]
  for (int i = threadIdx.x >> 2; i < c; i += kTmThreads >> 2)
    for (int j = threadIdx.x & 3; j < d; j += 4) cp_async_f64(&ms[i * d + j], M + (int64_t)i * ldm + j, true);
  const int rstep = kTmThreads / d, cstep = kTmThreads - (kTmThreads / d) * d;
  const int r_first = threadIdx.x / d, c_first = threadIdx.x - (threadIdx.x / d) * d;
  for (int64_t base = (int64_t)blockIdx.x * rpc; base < rows; base += (int64_t)gridDim.x * rpc) {
    const int nr = (int)imin64(rpc, rows - base);
    __syncthreads();  // the previous tile's reads of ts are done
    for (int rr = threadIdx.x >> 2; rr < nr; rr += kTmThreads >> 2) {
      const double* src = X + (base + rr) * ldx;
      for (int cc = threadIdx.x & 3; cc < c; cc += 4) cp_async_f64(&ts[rr * sp + cc], src + cc, true);
    }
    cp_async_wait_all();
    __syncthreads();
    int rr = r_first, cc = c_first;
    while (rr < nr) {
      // four elements per round: their beta * O reads are in flight together
      int er[4], ec[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        er[u] = rr;
        ec[u] = cc;
        rr += rstep;
        cc += cstep;
        if (cc >= d) {
          cc -= d;
          ++rr;
        }
      }
      double old[4], acc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        old[u] = (beta != 0.0 && er[u] < nr) ? O[(base + er[u]) * ldo + ec[u]] : 0.0;
        acc[u] = 0.0;
      }
      for (int i = 0; i < c; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (er[u] < nr) acc[u] = fma(ts[er[u] * sp + i], ms[i * d + ec[u]], acc[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (er[u] < nr) {
          const int64_t row = base + er[u];
          double v = alpha * acc[u];
          if (row < top_rows) v += top[row * ldt + ec[u]];
          O[row * ldo + ec[u]] = (beta == 0.0) ? v : fma(beta, old[u], v);
        }
      }
    }
  }
}

// Wide outputs (d > 32): one warp per row, lane q*32 + l owns output
// column l + 32 q (coalesced 256-byte stores), the row of X is loaded by
// lanes 0..c-1 and broadcast by shuffles, M is read from shared memory with
// consecutive lanes on consecutive columns.  Rows are visited grid-stride.
template <int QMAX>
__global__ void __launch_bounds__(kTmThreads)
tall_mul_wide_kernel(int64_t rows, int c, const double* X, int64_t ldx, int d, const double* __restrict__ M,
                     int64_t ldm, double alpha, double beta, double* O, int64_t ldo,
                     const double* __restrict__ top, int64_t ldt, int64_t top_rows) {
  extern __shared__ __align__(16) double tw_smem[];
  for (int i = threadIdx.x >> 5; i < c; i += kTmThreads >> 5)
    for (int j = threadIdx.x & 31; j < d; j += 32) tw_smem[i * d + j] = M[(int64_t)i * ldm + j];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (kTmThreads >> 5);
  int64_t row = (int64_t)blockIdx.x * (kTmThreads >> 5) + (threadIdx.x >> 5);
  // the next row of X is loaded while the current one is processed
  double nx0 = 0.0, nx1 = 0.0;
  if (row < rows) {
    nx0 = lane < c ? X[row * ldx + lane] : 0.0;
    nx1 = lane + 32 < c ? X[row * ldx + lane + 32] : 0.0;
  }
  for (; row < rows; row += nw) {
    const double x0 = nx0, x1 = nx1;
    if (row + nw < rows) {
      nx0 = lane < c ? X[(row + nw) * ldx + lane] : 0.0;
      nx1 = lane + 32 < c ? X[(row + nw) * ldx + lane + 32] : 0.0;
    }
    double* orow = O + row * ldo;
    double acc[QMAX], old[QMAX];
#pragma unroll
    for (int q = 0; q < QMAX; ++q) {
      acc[q] = 0.0;
      old[q] = (beta != 0.0 && lane + 32 * q < d) ? orow[lane + 32 * q] : 0.0;
    }
    for (int i = 0; i < c; ++i) {
      const double xi = __shfl_sync(0xffffffffu, i < 32 ? x0 : x1, i & 31);
      const double* mr = tw_smem + i * d + lane;
#pragma unroll
      for (int q = 0; q < QMAX; ++q)
        if (lane + 32 * q < d) acc[q] = fma(xi, mr[32 * q], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < QMAX; ++q) {
      const int j = lane + 32 * q;
      if (j < d) {
        double v = alpha * acc[q];
        if (row < top_rows) v += top[row * ldt + j];
        orow[j] = (beta == 0.0) ? v : fma(beta, old[q], v);
      }
    }
  }
}

// Narrow outputs (d <= 16) of long row counts: one thread per row, M
// broadcast from shared memory; each thread writes its row's d values.
__global__ void __launch_bounds__(kTmThreads)
tall_mul_narrow_kernel(int64_t rows, int c, const double* X, int64_t ldx, int d, const double* __restrict__ M,
                       int64_t ldm, double alpha, double beta, double* O, int64_t ldo,
                       const double* __restrict__ top, int64_t ldt, int64_t top_rows) {
  __shared__ double nm[64 * 16];
  for (int e = threadIdx.x; e < c * d; e += kTmThreads) nm[e] = M[(int64_t)(e / d) * ldm + (e % d)];
  __syncthreads();
  const int64_t nt = (int64_t)gridDim.x * kTmThreads;
  for (int64_t row = (int64_t)blockIdx.x * kTmThreads + threadIdx.x; row < rows; row += nt) {
    const double* xr = X + row * ldx;
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0;
    for (int i = 0; i < c; ++i) {
      const double xi = xr[i];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < d) acc[j] = fma(xi, nm[i * d + j], acc[j]);
    }
    double* orow = O + row * ldo;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j < d) {
        double v = alpha * acc[j];
        if (row < top_rows) v += top[row * ldt + j];
        orow[j] = (beta == 0.0) ? v : fma(beta, orow[j], v);
      }
    }
  }
}

int tall_mul(int64_t rows, int c, const double* X, int64_t ldx, int d, const double* M, int64_t ldm, double alpha,
             double beta, double* O, int64_t ldo, cudaStream_t s, const double* top, int64_t ldt,
             int64_t top_rows) {
  SPB_REQUIRE(c >= 1 && d >= 1 && c <= kTallMax && d <= 4 * kTallMax && c * d <= 64 * 64,
              "tall_mul supports c <= 64, d <= 256, c * d <= 4096");
  if (rows == 0) return SP_OK;
  static bool attr = false;
  if (!attr) {
    SPB_CUDA(cudaFuncSetAttribute(tall_mul_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    attr = true;
  }
  const int64_t tr = top ? top_rows : 0;
  if (rows >= 4096 && d > 32) {  // wide: warp per row
    const size_t smem = (size_t)c * d * sizeof(double);
    const int grid = (int)std::min<int64_t>(ceil_div(rows, kTmThreads / 32), 8 * kNumSMs);
#define SPB_TMW(Q)                                                                                          \
  do {                                                                                                      \
    static bool attr_w = false;                                                                             \
    if (!attr_w) {                                                                                          \
      SPB_CUDA(cudaFuncSetAttribute(tall_mul_wide_kernel<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                    64 * 1024));                                                            \
      attr_w = true;                                                                                        \
    }                                                                                                       \
    tall_mul_wide_kernel<Q><<<grid, kTmThreads, smem, s>>>(rows, c, X, ldx, d, M, ldm, alpha, beta, O, ldo, \
                                                           top, ldt, tr);                                   \
  } while (0)
    if (d <= 64)
      SPB_TMW(2);
    else if (d <= 128)
      SPB_TMW(4);
    else
      SPB_TMW(8);
#undef SPB_TMW
    count_launch();
    SPB_CHECK_LAUNCH();
    return SP_OK;
  }
  if (rows >= 65536 && d <= 16 && c * d <= 64 * 16) {  // narrow: thread per row
    const int grid = (int)std::min<int64_t>(ceil_div(rows, kTmThreads), 8 * kNumSMs);
    tall_mul_narrow_kernel<<<grid, kTmThreads, 0, s>>>(rows, c, X, ldx, d, M, ldm, alpha, beta, O, ldo, top, ldt,
                                                       tr);
    count_launch();
    SPB_CHECK_LAUNCH();
    return SP_OK;
  }
  // rows per CTA: 2048 outputs, bounded by the shared-memory opt-in (narrow
  // products -- d <= 4 with c = 64 -- asked for 268 KB and failed to launch)
  const int rpc_smem = (int)((size_t)(160 * 1024) / sizeof(double) - (size_t)c * d) / (c + 1);
  const int rpc = std::max(1, std::min(std::min(512, 2048 / d), rpc_smem));
  const size_t smem = ((size_t)c * d + (size_t)rpc * (c + 1)) * sizeof(double);
  const int grid = (int)std::min<int64_t>(ceil_div(rows, rpc), 8 * kNumSMs);
  SPB_CUDA(launch_pdl((tall_mul_kernel), dim3(grid), dim3(kTmThreads), smem, s, rows, c, X, ldx, d, M, ldm, alpha, beta, O, ldo, top, ldt,
                                                 top ? top_rows : 0, rpc));
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

}  // namespace spb
