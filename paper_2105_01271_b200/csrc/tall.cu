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
// to sp - 1 columns and up to `tile` rows).
__device__ __forceinline__ void stage_rows(double* s, int sp, int tile, const double* X, int64_t ldx,
                                           int64_t base, int nr, int c) {
  const int width = sp - 1;
  for (int e = threadIdx.x; e < tile * width; e += blockDim.x) {
    const int rr = e / width, cc = e - rr * width;
    const bool ok = rr < nr && cc < c;
    cp_async_f64(&s[rr * sp + cc], ok ? X + (base + rr) * ldx + cc : X, ok);
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

// O = alpha X M + beta O.  A CTA owns R = min(512, 2048 / d) consecutive rows
// and each thread forms output elements t, t + 256, ... of that row-major
// R x d block, so loads and stores are coalesced whatever d is; the rows of X
// and all of M are staged in shared memory (cp.async).  Each output row
// depends only on the same row of X, and the CTA's rows are staged before
// any output is written, so O may alias X (same rows, any columns).
constexpr int kTmThreads = 256;

__global__ void __launch_bounds__(kTmThreads)
tall_mul_kernel(int64_t rows, int c, const double* X, int64_t ldx, int d, const double* __restrict__ M,
                int64_t ldm, double alpha, double beta, double* O, int64_t ldo, const double* __restrict__ top,
                int64_t ldt, int64_t top_rows, int rpc) {
  extern __shared__ __align__(16) double tm_smem[];
  const int sp = c + 1;
  double* ms = tm_smem;          // [c][d]
  double* ts = tm_smem + c * d;  // [rpc][sp]
  const int64_t base = (int64_t)blockIdx.x * rpc;
  const int nr = (int)imin64(rpc, rows - base);
  for (int e = threadIdx.x; e < c * d; e += kTmThreads) {
    const int i = e / d, j = e - (e / d) * d;
    cp_async_f64(&ms[e], M + (int64_t)i * ldm + j, true);
  }
  for (int e = threadIdx.x; e < nr * c; e += kTmThreads) {
    const int rr = e / c, cc = e - (e / c) * c;
    cp_async_f64(&ts[rr * sp + cc], X + (base + rr) * ldx + cc, true);
  }
  cp_async_wait_all();
  __syncthreads();
  const int ne = nr * d;
  for (int e0 = threadIdx.x; e0 < ne; e0 += 4 * kTmThreads) {
    double acc[4], old[4];
    int rr[4], cc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * kTmThreads;
      rr[u] = e < ne ? e / d : 0;
      cc[u] = e < ne ? e - rr[u] * d : 0;
      acc[u] = 0.0;
      old[u] = (beta != 0.0 && e < ne) ? O[(base + rr[u]) * ldo + cc[u]] : 0.0;
    }
    for (int i = 0; i < c; ++i) {
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = fma(ts[rr[u] * sp + i], ms[i * d + cc[u]], acc[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * kTmThreads;
      if (e < ne) {
        const int64_t row = base + rr[u];
        double v = alpha * acc[u];
        if (row < top_rows) v += top[row * ldt + cc[u]];
        O[row * ldo + cc[u]] = (beta == 0.0) ? v : fma(beta, old[u], v);
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
  const int rpc = std::max(1, std::min(512, 2048 / d));
  const size_t smem = ((size_t)c * d + (size_t)rpc * (c + 1)) * sizeof(double);
  tall_mul_kernel<<<ceil_div(rows, rpc), kTmThreads, smem, s>>>(rows, c, X, ldx, d, M, ldm, alpha, beta, O, ldo,
                                                                top, ldt, top ? top_rows : 0, rpc);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

}  // namespace spb
