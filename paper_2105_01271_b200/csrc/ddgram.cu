// R factor of a tall block X (rows x b, b <= 32) by Cholesky of its Gram
// matrix accumulated and factored in double-double arithmetic (~106-bit
// significand): R^T R = X^T X.  Used for the Rayleigh-Ritz core of the
// sketch-side subspace iteration (svd_top, pipeline.cu), which needs R only
// (Z = C^T Q = P R, SVD of R^T) -- the role of thin_qr's R in
// src/kernels.py:62-84 / src/power.py:166-170.
//
// Why this is as accurate as Householder here: squaring X squares its
// condition number, which in FP64 would wipe out singular values below
// ~1e-8 sigma_1; in double-double the Gram keeps them down to ~1e-15 sigma_1
// (sigma^2 down to ~1e-30 of the trace, above the accumulated dd rounding),
// and rounding the dd Cholesky factor to FP64 is a column-wise relative
// perturbation of R, i.e. a backward error of ~eps ||X|| -- the Householder
// bound.  Pivots below kDgFloor * trace(G) (singular values below ~3e-15
// ||X||_F, i.e. the rounding floor of X itself) are set to zero with their
// row: the numerically rank-deficient tail of a subspace block.  Measured on
// the cfg2 sketch (tools/ in DESIGN.md sec. 4): top singular values and the
// kept subspace agree with the Householder R to 1e-16 sigma_1 / 1e-14 in
// angle.
//
// One launch: ~sqrt(rows) CTAs (<= 148) each accumulate a partial Gram of a
// contiguous row range over the 528 upper-triangle entries (rows staged 64 at
// a time through shared memory; error-free products by FMA, Neumaier-style
// compensated sums, two entries per thread); the partials are summed in dd
// in two fixed-order levels (the last CTA of each group of 8 by an atomic
// ticket, then the last group) -- bitwise reproducible -- and the last CTA factors
// the dd Gram right-looking in shared memory (pivot by an FP64 rsqrt with one
// dd Newton correction; the trailing update S_ik -= S_ji S_jk / d_j).  It
// replaces the 32-step Householder TSQR factor (tsqr.cu), whose per-column
// cluster-wide reductions are latency bound.
#include <cmath>
#include <map>
#include <mutex>

#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

namespace {

struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd dd_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd dd_quick(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
// accurate dd + dd
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = dd_two_sum(a.hi, b.hi);
  const dd t = dd_two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = dd_quick(s.hi, s.lo);
  s.lo += t.lo;
  return dd_quick(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  const double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e = fma(a.hi, b.lo, e);
  e = fma(a.lo, b.hi, e);
  return dd_quick(p, e);
}
// 1 / a (a.hi > 0): FP64 quotient plus one dd correction
__device__ __forceinline__ dd dd_recip(dd a) {
  const double q1 = 1.0 / a.hi;
  const dd r = dd_add({1.0, 0.0}, dd_neg(dd_mul(a, {q1, 0.0})));
  return dd_quick(q1, r.hi / a.hi);
}
__device__ __forceinline__ dd dd_sqrt(dd a) {
  const double x = sqrt(a.hi);
  const double p = x * x;
  const double e = fma(x, x, -p);
  const double r = ((a.hi - p) - e + a.lo) / (2.0 * x);
  return dd_quick(x, r);
}

constexpr int kDgB = 32;                         // block width (padded)
constexpr int kDgEnt = kDgB * (kDgB + 1) / 2;   // upper-triangle entries (528)
constexpr int kDgThreads = 288;                  // 2 entries per thread (9 warps)
constexpr int kDgTile = 64;                      // rows staged per step
constexpr double kDgFloor = 1e-29;               // pivot floor relative to trace(G)
constexpr int kDgGroup = 8;                      // partials per first-level group
constexpr int kDgTickets = 32;                   // 1 + max groups (148 / 8 -> 19)

// upper-triangle entry e -> (i, j), i <= j, row-major over the triangle
__device__ __forceinline__ void dg_entry(int e, int& i, int& j) {
  if (e >= kDgEnt) {  // padding threads
    i = j = 0;
    return;
  }
  int r = 0, base = 0;
  while (e >= base + (kDgB - r)) {
    base += kDgB - r;
    ++r;
  }
  i = r;
  j = r + (e - base);
}

// 1 / sqrt(d) in dd (d.hi > 0 normal): FP64 rsqrt, one dd Newton correction
__device__ __forceinline__ dd dd_rsqrt(dd d) {
  const double y = fast_range(d.hi) ? fast_rsqrt(d.hi) : 1.0 / sqrt(d.hi);
  const double y2 = y * y;
  const dd yy = {y2, fma(y, y, -y2)};
  const dd r = dd_add({1.0, 0.0}, dd_neg(dd_mul(d, yy)));  // 1 - d y^2, tiny
  return dd_quick(y, 0.5 * y * r.hi);
}

__global__ void __launch_bounds__(kDgThreads)
ddgram_chol_kernel(int64_t rows, int b, const double* __restrict__ X, int64_t ldx, int nslab, int64_t slab_stride,
                   int64_t rows_per_cta,
                   double2* __restrict__ partial, double2* __restrict__ gpart, int* __restrict__ ticket,
                   double* __restrict__ R, int64_t ldr) {
  SPB_TDECL;
  SPB_PDL_ENTRY();
  SPB_TMARK(0);
  __shared__ __align__(16) double xs[kDgTile][kDgB + 1];
  __shared__ dd S[kDgB][kDgB + 1];
  __shared__ double piv_r[2];  // 1 / r_jj, double-buffered over steps
  __shared__ dd piv_d[2];      // 1 / d_j
  __shared__ int last;
  const int t = threadIdx.x;
  int ei[2], ej[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) dg_entry(2 * t + u, ei[u], ej[u]);
  // Neumaier-style accumulation with error-free products: hi + lo, lo
  // collecting the rounding errors (|lo| stays ~n eps |hi|); even and odd rows
  // in separate accumulators (two independent dependency chains per entry)
  double hi[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, lo[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = imin64(rows, r0 + rows_per_cta);
  for (int64_t c0 = r0; c0 < r1; c0 += kDgTile) {
    const int nr = (int)imin64(kDgTile, r1 - c0);
    if (nslab == 1) {
      for (int e = t; e < kDgTile * kDgB; e += kDgThreads) {
        const int rr = e / kDgB, cc = e % kDgB;
        const bool ok = rr < nr && cc < b;
        cp_async_f64(&xs[rr][cc], ok ? X + (c0 + rr) * ldx + cc : X, ok);
      }
      cp_async_wait_all();
    } else {  // X = sum of the split-K slabs, in slab order
      for (int e = t; e < kDgTile * kDgB; e += kDgThreads) {
        const int rr = e / kDgB, cc = e % kDgB;
        double v = 0.0;
        if (rr < nr && cc < b) {
          const double* p = X + (c0 + rr) * ldx + cc;
          v = __ldcg(p);
#pragma unroll 4
          for (int q = 1; q < nslab; ++q) v += __ldcg(p + (int64_t)q * slab_stride);
        }
        xs[rr][cc] = v;
      }
    }
    __syncthreads();
    if (c0 == r0) SPB_TMARK(1);
    if (2 * t < kDgEnt) {
#pragma unroll 2
      for (int rr = 0; rr < kDgTile; rr += 2) {  // rows >= nr were zero-filled
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const double xi = xs[rr + h][ei[u]], xj = xs[rr + h][ej[u]];
            const double p = xi * xj;
            const double pe = fma(xi, xj, -p);
            const double sm = hi[h][u] + p;
            const double bb = sm - hi[h][u];
            lo[h][u] += ((hi[h][u] - (sm - bb)) + (p - bb)) + pe;
            hi[h][u] = sm;
          }
      }
    }
    __syncthreads();
  }
  if (2 * t < kDgEnt) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const dd a = dd_add(dd_quick(hi[0][u], lo[0][u]), dd_quick(hi[1][u], lo[1][u]));
      partial[(int64_t)blockIdx.x * kDgEnt + 2 * t + u] = make_double2(a.hi, a.lo);
    }
  }
  // ---- two-level fixed-order reduction: the last CTA of each group of
  // kDgGroup CTAs sums the group's partials (in CTA order), the last group
  // sums the group totals (in group order) and factors
  SPB_TMARK(2);
  const int nb = (int)gridDim.x, ngrp = (nb + kDgGroup - 1) / kDgGroup;
  const int grp = (int)blockIdx.x / kDgGroup, g0 = grp * kDgGroup;
  const int gsz = nb - g0 < kDgGroup ? nb - g0 : kDgGroup;
  __threadfence();
  __syncthreads();
  if (t == 0) last = atomicAdd(ticket + 1 + grp, 1) == gsz - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  auto sum_rows = [&](const double2* src, int first, int count, dd (&g)[2]) {
    double2 v[kDgGroup][2];
#pragma unroll
    for (int q = 0; q < kDgGroup; ++q)
#pragma unroll
      for (int u = 0; u < 2; ++u)
        v[q][u] = q < count ? __ldcg(src + (int64_t)(first + q) * kDgEnt + 2 * t + u) : make_double2(0.0, 0.0);
    g[0] = g[1] = {0.0, 0.0};
#pragma unroll
    for (int q = 0; q < kDgGroup; ++q)
      if (q < count)
#pragma unroll
        for (int u = 0; u < 2; ++u) g[u] = dd_add(g[u], {v[q][u].x, v[q][u].y});
  };
  if (2 * t < kDgEnt) {
    dd g[2];
    sum_rows(partial, g0, gsz, g);
#pragma unroll
    for (int u = 0; u < 2; ++u) gpart[(int64_t)grp * kDgEnt + 2 * t + u] = make_double2(g[u].hi, g[u].lo);
  }
  __threadfence();
  __syncthreads();
  if (t == 0) {
    ticket[1 + grp] = 0;
    last = atomicAdd(ticket, 1) == ngrp - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  SPB_TMARK(3);
  if (2 * t < kDgEnt) {
    dd g[2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int c0 = 0; c0 < ngrp; c0 += kDgGroup) {
      dd h[2];
      sum_rows(gpart, c0, ngrp - c0 < kDgGroup ? ngrp - c0 : kDgGroup, h);
#pragma unroll
      for (int u = 0; u < 2; ++u) g[u] = dd_add(g[u], h[u]);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) S[ei[u]][ej[u]] = g[u];
  }
  __syncthreads();
  SPB_TMARK(4);
  double tr = 0.0;
  for (int j = 0; j < b; ++j) tr += S[j][j].hi;
  const double floor_abs = kDgFloor * tr;
  // right-looking Cholesky of the upper triangle; thread (gi, 4 columns).
  // The pivot of step j + 1 is formed by the owner of S[j+1][j+1] from its
  // freshly updated register value (double-buffered), so a step costs one
  // barrier.  Pivot data: 1 / r_jj in FP64 (it only scales R's row j, which
  // is rounded to FP64 anyway) and 1 / d_j in dd (the trailing update).
  const int gi = t >> 3, j0 = (t & 7) * 4;
  const bool chol_thread = t < 256;
  auto pivot = [&](dd d, int buf) {
    if (d.hi > floor_abs && d.hi < 1e300) {
      const bool fr = fast_range(d.hi);
      piv_r[buf] = fr ? fast_rsqrt(d.hi) : 1.0 / sqrt(d.hi);
      const double q1 = fr ? fast_rcp(d.hi) : 1.0 / d.hi;
      const double p = d.hi * q1;
      const double e = fma(d.hi, q1, -p);
      const double r = fma(-d.lo, q1, (1.0 - p) - e);  // 1 - d q1 (1 - p exact)
      piv_d[buf] = dd_quick(q1, r * q1);
    } else {
      piv_r[buf] = 0.0;
      piv_d[buf] = {0.0, 0.0};
    }
  };
  if (t == 0) pivot(S[0][0], 0);
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    const double rinv = piv_r[j & 1];
    const dd inv2 = piv_d[j & 1];
    // R row j: R_jk = S_jk / r_jj (k >= j), zeros below the diagonal
    if (chol_thread && gi == j) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = j0 + u;
        if (k < b) R[(int64_t)j * ldr + k] = k >= j ? S[j][k].hi * rinv : 0.0;
      }
    }
    // trailing update S_ik -= S_ji S_jk / d_j (i <= k).  Step j reads row j
    // only and writes rows > j: no barrier between the two.
    if (chol_thread && gi > j && gi < b) {
      dd rowj[4], mine[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        rowj[u] = S[j][j0 + u];
        mine[u] = S[gi][j0 + u];
      }
      if (inv2.hi != 0.0) {
        const dd f = dd_mul(S[j][gi], inv2);
#pragma unroll
        for (int u = 0; u < 4; ++u) mine[u] = dd_add(mine[u], dd_neg(dd_mul(f, rowj[u])));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = j0 + u;
          if (k >= gi && k < b) S[gi][k] = mine[u];
        }
      }
      if (gi == j + 1 && j0 <= gi && gi < j0 + 4) {
        dd dnext = mine[0];
#pragma unroll
        for (int u = 1; u < 4; ++u)
          if (j0 + u == gi) dnext = mine[u];
        pivot(dnext, (j + 1) & 1);
      }
    }
    __syncthreads();
  }
  SPB_TMARK(5);
  if (t == 0) {
    *ticket = 0;
#ifdef SPB_PHASE_TRACE
    SPB_TPRINT("ddgram load|acc|wait|reduce|chol", 6);
#endif
  }
}

// Per-(device, stream) ticket words {final, group 0..}: zeroed once, each
// reset by the CTA that consumes it.
static int dd_ticket(cudaStream_t s, int** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, int*> words;
  int dev = 0;
  SPB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = words.find({dev, s});
  if (it == words.end()) {
    int* p = nullptr;
    SPB_CUDA(cudaMalloc(&p, kDgTickets * sizeof(int)));
    SPB_CUDA(cudaMemsetAsync(p, 0, kDgTickets * sizeof(int), s));
    it = words.emplace(std::make_pair(dev, s), p).first;
  }
  *out = it->second;
  return SP_OK;
}

}  // namespace

bool gram_chol_dd_ok(int64_t rows, int b) { return b >= 1 && b <= kDgB && rows >= b; }

// R (b x b upper, ld ldr; zeros below the diagonal) with
// R^T R = X^T X, X rows x b (ld ldx), or X = the sum of nslab split-K slabs
// slab_stride apart (summed in slab order while the tiles are staged).
// Asynchronous.
int gram_chol_dd(int64_t rows, int b, const double* X, int64_t ldx, double* R, int64_t ldr, Arena& ar,
                 cudaStream_t s, int nslab, int64_t slab_stride) {
  SPB_REQUIRE(gram_chol_dd_ok(rows, b), "gram_chol_dd: shape out of range");
  int* ticket = nullptr;
  SPB_TRY(dd_ticket(s, &ticket));
  // ~one tile per CTA for small blocks, at most one CTA per SM
  // partials ~ sqrt(rows): the per-CTA accumulation and the last CTA's sum
  // of the partials then take about the same time; at most one CTA per SM
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(kNumSMs, (int64_t)std::sqrt((double)rows)));
  const int64_t per = ceil_div(rows, ctas);
  const int nb = (int)ceil_div(rows, per);
  double2* part = ar.alloc<double2>((size_t)(nb + (nb + kDgGroup - 1) / kDgGroup) * kDgEnt);
  if (!part) {
    set_error("gram_chol_dd workspace allocation failed");
    return SP_ECUDA;
  }
  double2* gpart = part + (size_t)nb * kDgEnt;
  SPB_CUDA(launch_pdl((ddgram_chol_kernel), dim3(nb), dim3(kDgThreads), 0, s, rows, b, X, ldx, std::max(1, nslab),
                      slab_stride, per, part, gpart,
                      ticket, R, ldr));
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

}  // namespace spb
