// K5: one-sided (Hestenes) Jacobi SVD of a small square core, one CTA.
//
// Replaces the LAPACK gesdd behind thin_svd (src/kernels.py:87-94) for the
// sketch-sized cores (R factors of TSQR, <= 256 columns).  One-sided Jacobi
// is backward stable and computes small singular values of graded matrices to
// high RELATIVE accuracy, which is what the 1e-12 kept-rank cut
// (src/kernels.py:19, 158-168) needs.
//
// Columns are paired with the round-robin (circle) schedule: each round
// rotates n/2 disjoint pairs, one warp per pair, rows across the lanes.
// The working matrix W and the accumulated rotations V live in shared memory
// when they fit (n <= 112) and in a global scratch otherwise.  Convergence:
// a sweep with no rotation (|w_p.w_q| <= 1e-15 ||w_p|| ||w_q|| for every pair).
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace cg = cooperative_groups;

namespace spb {

constexpr int kJacMaxSweeps = 40;
constexpr double kJacTol = 1e-15;
constexpr double kJacQuad = 1e-8;
// Stopping rule.  A sweep whose rotated couplings g / sqrt(a b) were all below kJacQuad leaves
// only ~kJacQuad^2-sized ones behind when the singular values are separated (cyclic Jacobi
// converges quadratically), so it is the last -- UNLESS the sweep contained a large-angle
// rotation: inside a cluster of (nearly) equal singular values the angle is not small however
// small the coupling, the two columns' couplings to everything else are mixed, not squared, and
// what the sweep leaves behind is as large as what it started from (flat stretches of the
// spectrum were left with 1-4e-9 of non-orthogonality in U; found by scripts/fuzz_api.py).  Such
// a sweep is the last only once all its couplings were below kJacFloor.  Per-sweep flag bits:
constexpr double kJacFloor = 1e-11;
constexpr double kJacSin2 = 1e-8;  // sin^2(2 theta) above which a rotation counts as large-angle
constexpr int kJfAny = 1, kJfQuad = 2, kJfFloor = 4, kJfWide = 8;
__host__ __device__ __forceinline__ bool jac_continue(int flags) {
  return (flags & kJfQuad) || ((flags & kJfFloor) && (flags & kJfWide));
}

__device__ __forceinline__ void rr_pair(int np, int round, int k, int& p, int& q) {
  const int N1 = np - 1;
  if (k == 0) {
    p = 0;
    q = 1 + (round % N1);
  } else {
    p = 1 + ((round + k) % N1);
    q = 1 + ((round - k + N1) % N1);
  }
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

// W, Vm: column-major np x np (column c at c*np)
__global__ void __launch_bounds__(1024)
jacobi_kernel(int n, int np, const double* __restrict__ M, int64_t ldm, double* __restrict__ U,
              int64_t ldu, double* __restrict__ S, double* __restrict__ Vout, int64_t ldv,
              double* gW, double* gV, bool use_smem) {
  extern __shared__ double dyn[];
  __shared__ int rot_count;
  __shared__ double sig_s[256];
  double* W = use_smem ? dyn : gW;
  double* Vm = use_smem ? dyn + np * np : gV;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nthr >> 5;
  __shared__ double fro_part[32];
  double fro = 0.0;
  for (int e = tid; e < np * np; e += nthr) {
    const int c = e / np, i = e % np;
    const double x = (i < n && c < n) ? M[(int64_t)i * ldm + c] : 0.0;
    W[e] = x;
    fro = fma(x, x, fro);
    Vm[e] = (i == c) ? 1.0 : 0.0;
  }
  fro = warp_sum(fro);
  if (lane == 0) fro_part[warp] = fro;
  __syncthreads();
  fro = 0.0;
  for (int w = 0; w < nwarps; ++w) fro += fro_part[w];
  // Columns below 1e-15 ||M||_F are rounding noise: they are left out of the
  // rotation schedule altogether (their singular values are below any cut the
  // path uses), so a rank-17 core of width 32 runs the tournament on 18
  // columns instead of 32.
  const double negl = 1e-30 * fro;
  __shared__ int act[256];
  __shared__ int nact_s;
  for (int c = warp; c < np; c += nwarps) {
    double a = 0.0;
    for (int i = lane; i < np; i += 32) a = fma(W[c * np + i], W[c * np + i], a);
    a = warp_sum(a);
    if (lane == 0) sig_s[c] = a;
  }
  __syncthreads();
  if (tid == 0) {
    int na = 0;
    for (int c = 0; c < n; ++c)
      if (sig_s[c] > negl) act[na++] = c;
    if (na & 1) act[na++] = -1;  // pad to even
    nact_s = na;
  }
  __syncthreads();
  const int na = nact_s;
  __shared__ unsigned long long relmax_bits;  // largest |g| / sqrt(a b) rotated this sweep
  for (int sweep = 0; sweep < kJacMaxSweeps && na >= 2; ++sweep) {
    if (tid == 0) {
      rot_count = 0;
      relmax_bits = 0ull;
    }
    __syncthreads();
    for (int round = 0; round < na - 1; ++round) {
      for (int k = warp; k < na / 2; k += nwarps) {
        int pi, qi;
        rr_pair(na, round, k, pi, qi);
        int p = act[pi], q = act[qi];
        if (p < 0 || q < 0) continue;
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        double* wp = W + p * np;
        double* wq = W + q * np;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int i = lane; i < np; i += 32) {
          const double x = wp[i], y = wq[i];
          a = fma(x, x, a);
          b = fma(y, y, b);
          g = fma(x, y, g);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        g = warp_sum(g);
        if (g != 0.0 && fmin(a, b) > negl && fabs(g) > kJacTol * sqrt(a) * sqrt(b)) {
          const double zeta = (b - a) / (2.0 * g);
          double t;
          if (fabs(zeta) > 1e150)
            t = 0.5 / zeta;
          else
            t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
          const double c = 1.0 / sqrt(fma(t, t, 1.0));
          const double s = c * t;
          double* vp = Vm + p * np;
          double* vq = Vm + q * np;
          for (int i = lane; i < np; i += 32) {
            const double x = wp[i], y = wq[i];
            wp[i] = c * x - s * y;
            wq[i] = fma(s, x, c * y);
            const double u = vp[i], w = vq[i];
            vp[i] = c * u - s * w;
            vq[i] = fma(s, u, c * w);
          }
          if (lane == 0) {
            atomicAdd(&rot_count, 1);
            atomicMax(&relmax_bits, (unsigned long long)__double_as_longlong(fabs(g) / (sqrt(a) * sqrt(b))));
          }
        }
      }
      __syncthreads();
    }
    // quadratic convergence: a sweep whose rotations were all below kJacQuad
    // in relative size leaves only ~kJacQuad^2-sized ones for the next, which
    // would only confirm convergence (the jacobi32 rule)
    if (rot_count == 0 || __longlong_as_double((long long)relmax_bits) < kJacFloor) break;  // (no quadratic shortcut here)
    __syncthreads();
  }
  // singular values = column norms, sorted descending (stable by index)
  for (int c = warp; c < np; c += nwarps) {
    double a = 0.0;
    for (int i = lane; i < np; i += 32) a = fma(W[c * np + i], W[c * np + i], a);
    a = warp_sum(a);
    if (lane == 0) sig_s[c] = sqrt(a);
  }
  __syncthreads();
  for (int c = warp; c < n; c += nwarps) {
    const double sc = sig_s[c];
    int rank = 0;
    for (int d = lane; d < np; d += 32) {
      const double sd = sig_s[d];
      rank += (sd > sc || (sd == sc && d < c)) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (rank >= n) continue;  // a padding column outranks it only if all else is zero
    if (lane == 0) S[rank] = sc;
    const double inv = sc > 0.0 ? 1.0 / sc : 0.0;
    for (int i = lane; i < n; i += 32) {
      U[(int64_t)i * ldu + rank] = W[c * np + i] * inv;
      Vout[(int64_t)i * ldv + rank] = Vm[c * np + i];
    }
  }
}

// ---------------------------------------------------------- n <= 32 ----
// LANE = COLUMN variant for the cores of the path (b <= 32): warp w holds
// rows [8w, 8w + 8) of every column, lane c column c, so a pair's partner
// column arrives by 8 shuffles per warp and the three dot products are one
// 4-way shared-memory reduction (one __syncthreads per round, double
// buffered).  Both lanes of a pair compute the same rotation from the same
// sums in the same order (bitwise identical).  The rotation uses
//   t = sign(d) h / (|d| + hypot(d, h)),  d = b - a,  h = 2 g,
//   c = 1 / sqrt(1 + t^2),  s = c t
// (the tan(theta) root of t^2 + 2 (d/h) t - 1 = 0 of the classical formula).
constexpr int kJ32Warps = 4;

// circle-method partner of position x among na (even) players in round r
__device__ __forceinline__ int rr_partner(int x, int r, int na) {
  const int n1 = na - 1;
  if (x == 0) return 1 + (r % n1);
  int y = (2 * r - (x - 1)) % n1;
  if (y < 0) y += n1;
  y += 1;
  return y == x ? 0 : y;
}

// fixed-order sum of the NW warp partials of lane c
template <int NW>
__device__ __forceinline__ double jsum(const double (*p)[32], int c) {
  if constexpr (NW == 1) return p[0][c];
  if constexpr (NW == 2) return p[0][c] + p[1][c];
  return (p[0][c] + p[1][c]) + (p[2][c] + p[3][c]);
}

// NW warps x RPW rows (NW * RPW >= n); NW = 1 needs no block barrier in the
// rounds (the n <= 8 cores of the finish stage)
template <int NW, int RPW>
__global__ void __launch_bounds__(NW * 32)
jacobi32_kernel(int n, const double* __restrict__ M, int64_t ldm, double* __restrict__ U, int64_t ldu,
                double* __restrict__ S, double* __restrict__ Vout, int64_t ldv, bool trans, int64_t bsM = 0,
                int64_t bsU = 0, int64_t bsS = 0, int64_t bsV = 0) {
  SPB_PDL_ENTRY();
  // batched launches (block Jacobi): CTA b works on the b-th core
  M += blockIdx.x * bsM;
  U += blockIdx.x * bsU;
  S += blockIdx.x * bsS;
  if (Vout) Vout += blockIdx.x * bsV;
  __shared__ double part[2][NW][32][2];
  __shared__ double nrm_s[NW][32];
  __shared__ double sig_s[32];
  __shared__ int act[32], pos_s[32];
  __shared__ int na_s;
  const int w = threadIdx.x >> 5, c = threadIdx.x & 31;
  const bool want_v = Vout != nullptr;
  double x[RPW], v[RPW];
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int i = w * RPW + k;
    x[k] = (i < n && c < n) ? (trans ? M[(int64_t)c * ldm + i] : M[(int64_t)i * ldm + c]) : 0.0;
    v[k] = (i == c) ? 1.0 : 0.0;
  }
  // column norms and ||M||_F^2 (fixed order)
  double a0 = 0.0;
#pragma unroll
  for (int k = 0; k < RPW; ++k) a0 = fma(x[k], x[k], a0);
  nrm_s[w][c] = a0;
  __syncthreads();
  if (threadIdx.x == 0) {
    double fro = 0.0;
    double cn[32];
    for (int cc = 0; cc < 32; ++cc) {
      cn[cc] = jsum<NW>(nrm_s, cc);
      fro += cn[cc];
    }
    // columns below 1e-15 ||M||_F are rounding noise: left out of the schedule
    const double negl = 1e-30 * fro;
    int na = 0;
    for (int cc = 0; cc < 32; ++cc) pos_s[cc] = -1;
    for (int cc = 0; cc < n; ++cc)
      if (cn[cc] > negl) {
        pos_s[cc] = na;
        act[na++] = cc;
      }
    if (na & 1) act[na++] = -1;  // pad to even
    na_s = na;
  }
  __syncthreads();
  const int na = na_s, mypos = pos_s[c];
  // the circle-method schedule, once: ptab[round][lane] = partner lane or -1
  __shared__ signed char ptab[31][32];
  for (int e = threadIdx.x; e < (na - 1) * 32; e += blockDim.x) {
    const int rd = e >> 5, ln = e & 31, ps = pos_s[ln];
    ptab[rd][ln] = (signed char)(ps >= 0 ? act[rr_partner(ps, rd, na)] : -1);
  }
  __syncthreads();
  double fro2 = 0.0;
  for (int cc = 0; cc < 32; ++cc) fro2 += jsum<NW>(nrm_s, cc);
  const double negl = 1e-30 * fro2;
  int buf = 0;
  for (int sweep = 0; sweep < kJacMaxSweeps && na >= 2; ++sweep) {
    int rotated = 0;
    for (int round = 0; round < na - 1; ++round) {
      const int plane = ptab[round][c];
      const int src = plane >= 0 ? plane : c;
      double y[RPW], z[RPW];
#pragma unroll
      for (int k = 0; k < RPW; ++k) y[k] = __shfl_sync(0xffffffffu, x[k], src);
      if (want_v) {  // uniform across the CTA
#pragma unroll
        for (int k = 0; k < RPW; ++k) z[k] = __shfl_sync(0xffffffffu, v[k], src);
      }
      double pa0 = x[0] * x[0], pa1 = x[1] * x[1], pg0 = x[0] * y[0], pg1 = x[1] * y[1];
#pragma unroll
      for (int k = 2; k < RPW; k += 2) {
        pa0 = fma(x[k], x[k], pa0);
        pa1 = fma(x[k + 1], x[k + 1], pa1);
        pg0 = fma(x[k], y[k], pg0);
        pg1 = fma(x[k + 1], y[k + 1], pg1);
      }
      double a, g;
      if constexpr (NW == 1) {
        a = pa0 + pa1;
        g = pg0 + pg1;
      } else {
        part[buf][w][c][0] = pa0 + pa1;
        part[buf][w][c][1] = pg0 + pg1;
        __syncthreads();
        double ta[NW], tg[NW];
#pragma unroll
        for (int q = 0; q < NW; ++q) {
          ta[q] = part[buf][q][c][0];
          tg[q] = part[buf][q][c][1];
        }
        if constexpr (NW == 2) {
          a = ta[0] + ta[1];
          g = tg[0] + tg[1];
        } else {
          a = (ta[0] + ta[1]) + (ta[2] + ta[3]);
          g = (tg[0] + tg[1]) + (tg[2] + tg[3]);
        }
      }
      const double b = __shfl_sync(0xffffffffu, a, src);
      buf ^= 1;
      if (plane < 0) continue;
      const bool low = c < plane;  // canonical (p, q) = (min, max)
      const double ap = low ? a : b, aq = low ? b : a;
      const double apq = ap * aq;
      const bool big = !(apq < 1e300);  // rare: fall back to the overflow-safe forms
      if (!(g != 0.0 && fmin(ap, aq) > negl &&
            (big ? fabs(g) > kJacTol * sqrt(ap) * sqrt(aq) : g * g > (kJacTol * kJacTol) * apq)))
        continue;
      const double d = aq - ap, h = 2.0 * g;
      const double ad = fabs(d), ah = fabs(h);
      double cs, sn;
      bool wide;  // large-angle rotation (a cluster of equal singular values)
      if (ad < 1e140 && ah < 1e140 && (ad > 1e-140 || ah > 1e-140)) {
        // fast path, two dependent MUFU rsqrt (+ Newton) stages: rh =
        // 1 / hypot(d, h) gives cos 2theta = |d| rh and sin 2theta = h rh
        // (|theta| <= pi / 4); cs = sqrt((1 + cos 2theta) / 2) and
        // sn = sin 2theta / (2 cs) share one rsqrt of u in [1/2, 1]
        const double s2 = fma(d, d, h * h);
        const double rh = fast_rsqrt(s2);
        const double u = fma(0.5 * ad, rh, 0.5);
        const double w = fast_rsqrt(u);
        cs = u * w;
        sn = (copysign(0.5, d) * h) * (rh * w);
        wide = h * h > kJacSin2 * s2;
      } else {
        const double t = copysign(1.0, d) * h / (ad + hypot(d, h));
        cs = rsqrt(fma(t, t, 1.0));
        sn = cs * t;
        wide = fabs(t) > 5e-5;
      }
      // p' = cs p - sn q ; q' = sn p + cs q
      const double so = low ? -sn : sn;
#pragma unroll
      for (int k = 0; k < RPW; ++k) x[k] = fma(so, y[k], cs * x[k]);
      if (want_v) {
#pragma unroll
        for (int k = 0; k < RPW; ++k) v[k] = fma(so, z[k], cs * v[k]);
      }
      // a rotation of relative size above kJacQuad keeps the sweeps going
      if (big ? fabs(g) > kJacQuad * sqrt(ap) * sqrt(aq) : g * g > (kJacQuad * kJacQuad) * apq) rotated |= kJfQuad;
      if (big ? fabs(g) > kJacFloor * sqrt(ap) * sqrt(aq) : g * g > (kJacFloor * kJacFloor) * apq) rotated |= kJfFloor;
      if (wide) rotated |= kJfWide;
    }
    // Stop after a sweep whose rotations were all below kJacQuad in relative
    // size: cyclic Jacobi converges quadratically, so what the next sweep
    // would still find is ~n kJacQuad^2 / (relative gap) ~ 1e-15 of
    // ||w_p|| ||w_q|| (the kJacTol level: column changes ~1e-15, singular
    // values unchanged to second order) -- it is not run (5 -> 4 sweeps on
    // the cfg2 core).
    // (__syncthreads_or returns a truth value, not the OR of the bits: one vote per flag)
    const int fq = __syncthreads_or(rotated & kJfQuad) ? kJfQuad : 0;
    const int ff = __syncthreads_or(rotated & kJfFloor) ? kJfFloor : 0;
    const int fw = __syncthreads_or(rotated & kJfWide) ? kJfWide : 0;
    if (!jac_continue(fq | ff | fw)) {
#ifdef SPB_JACOBI_TRACE
      if (threadIdx.x == 0) printf("jacobi32 n=%d na=%d sweeps=%d\n", n, na, sweep + 1);
#endif
      break;
    }
  }
  // singular values = column norms, sorted descending (stable by index)
  double a1 = 0.0;
#pragma unroll
  for (int k = 0; k < RPW; ++k) a1 = fma(x[k], x[k], a1);
  nrm_s[w][c] = a1;
  __syncthreads();
  if (w == 0) sig_s[c] = sqrt(jsum<NW>(nrm_s, c));
  __syncthreads();
  const double sc = sig_s[c];
  int rank = 0;
  for (int d = 0; d < 32; ++d) {
    const double sd = sig_s[d];
    rank += (sd > sc || (sd == sc && d < c)) ? 1 : 0;
  }
  if (rank >= n) return;
  if (w == 0) S[rank] = sc;
  const double inv = sc > 0.0 ? 1.0 / sc : 0.0;
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int i = w * RPW + k;
    if (i < n) {
      U[(int64_t)i * ldu + rank] = x[k] * inv;
      if (want_v) Vout[(int64_t)i * ldv + rank] = v[k];
    }
  }
}

// ------------------------------------------------------- n > 112, grid ----
// W and V (column-major, n_p x n_p) do not fit in one SM's shared memory, so
// the rounds are spread over a cooperative grid: one warp per column pair
// (n_p / 2 pairs), W / V in global memory (L2-resident up to n ~ 2500), one
// grid barrier per round.  Used for the sketch cores (n <= 256) and for the
// size-general thin_svd of the drop-in (n up to the sketch widths, 16384);
// columns below 1e-15 ||M||_F never enter the schedule, so a numerically
// low-rank M (the BASELINE sketches) costs rounds only for its rank.  Every CTA derives the same active-column list
// from the same column norms; rotations, convergence test and sorting are
// those of the single-CTA kernel.
constexpr int kJgThreads = 128;

__global__ void __launch_bounds__(kJgThreads)
jacobi_grid_kernel(int n, int np, const double* __restrict__ M, int64_t ldm, bool trans, double* __restrict__ U,
                   int64_t ldu, double* __restrict__ S, double* __restrict__ Vout, int64_t ldv,
                   double* __restrict__ W, double* __restrict__ Vm, double* __restrict__ cn, int* rot,
                   unsigned long long* relmax) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ int act[];  // np entries (dynamic: n is not capped at 256)
  __shared__ int na_s;
  const int lane = threadIdx.x & 31;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gthr = (int64_t)gridDim.x * blockDim.x;
  const int gwarp = (int)(gtid >> 5), nwarps = (int)(gthr >> 5);
  for (int64_t e = gtid; e < (int64_t)np * np; e += gthr) {
    const int c = (int)(e / np), i = (int)(e % np);
    W[e] = (i < n && c < n) ? (trans ? M[(int64_t)c * ldm + i] : M[(int64_t)i * ldm + c]) : 0.0;
    Vm[e] = (i == c) ? 1.0 : 0.0;
  }
  if (gtid < 2) {
    rot[gtid] = 0;
    relmax[gtid] = 0ull;
  }
  grid.sync();
  for (int c = gwarp; c < np; c += nwarps) {
    double a = 0.0;
    for (int i = lane; i < np; i += 32) a = fma(W[(int64_t)c * np + i], W[(int64_t)c * np + i], a);
    a = warp_sum(a);
    if (lane == 0) cn[c] = a;
  }
  grid.sync();
  double fro = 0.0;
  for (int c = 0; c < np; ++c) fro += cn[c];
  const double negl = 1e-30 * fro;
  if (threadIdx.x == 0) {
    int na = 0;
    for (int c = 0; c < n; ++c)
      if (cn[c] > negl) act[na++] = c;
    if (na & 1) act[na++] = -1;
    na_s = na;
  }
  __syncthreads();
  const int na = na_s;
  for (int sweep = 0; sweep < kJacMaxSweeps && na >= 2; ++sweep) {
    for (int round = 0; round < na - 1; ++round) {
      if (round == 1 && gtid == 0) {  // nobody reads the other parity until this sweep ends
        rot[(sweep + 1) & 1] = 0;
        relmax[(sweep + 1) & 1] = 0ull;
      }
      for (int k = gwarp; k < na / 2; k += nwarps) {
        int pi, qi;
        rr_pair(na, round, k, pi, qi);
        int p = act[pi], q = act[qi];
        if (p < 0 || q < 0) continue;
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        double* wp = W + (int64_t)p * np;
        double* wq = W + (int64_t)q * np;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int i = lane; i < np; i += 32) {
          const double x = wp[i], y = wq[i];
          a = fma(x, x, a);
          b = fma(y, y, b);
          g = fma(x, y, g);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        g = warp_sum(g);
        // thresholds on squares and the MUFU-rsqrt rotation of jacobi32 (the
        // IEEE sqrt / division forms cost ~3000 dependent cycles per round)
        const double ab = a * b;
        const bool big = !(ab < 1e300);
        if (g != 0.0 && fmin(a, b) > negl &&
            (big ? fabs(g) > kJacTol * sqrt(a) * sqrt(b) : g * g > (kJacTol * kJacTol) * ab)) {
          const double d = b - a, h = 2.0 * g;
          const double ad = fabs(d), ah = fabs(h);
          double cs, sn;
          bool wide;  // large-angle rotation (see kJacFloor)
          if (ad < 1e140 && ah < 1e140 && (ad > 1e-140 || ah > 1e-140)) {
            const double s2 = fma(d, d, h * h);
            const double rh = fast_rsqrt(s2);
            const double u = fma(0.5 * ad, rh, 0.5);
            const double w = fast_rsqrt(u);
            cs = u * w;
            sn = (copysign(0.5, d) * h) * (rh * w);
            wide = h * h > kJacSin2 * s2;
          } else {
            const double t = copysign(1.0, d) * h / (ad + hypot(d, h));
            cs = rsqrt(fma(t, t, 1.0));
            sn = cs * t;
            wide = fabs(t) > 5e-5;
          }
          double* vp = Vm + (int64_t)p * np;
          double* vq = Vm + (int64_t)q * np;
          for (int i = lane; i < np; i += 32) {
            const double x = wp[i], y = wq[i];
            wp[i] = cs * x - sn * y;
            wq[i] = fma(sn, x, cs * y);
            const double u = vp[i], w = vq[i];
            vp[i] = cs * u - sn * w;
            vq[i] = fma(sn, u, cs * w);
          }
          if (lane == 0) {
            int fl = kJfAny | (wide ? kJfWide : 0);
            if (big ? fabs(g) > kJacQuad * sqrt(a) * sqrt(b) : g * g > (kJacQuad * kJacQuad) * ab) fl |= kJfQuad;
            if (big ? fabs(g) > kJacFloor * sqrt(a) * sqrt(b) : g * g > (kJacFloor * kJacFloor) * ab) fl |= kJfFloor;
            atomicOr(&rot[sweep & 1], fl);
          }
        }
      }
      grid.sync();
    }
    // same values in every thread after the barrier; the quadratic-convergence
    // stop of the single-CTA kernels
    if (!jac_continue(*(volatile int*)&rot[sweep & 1])) break;
  }
  // singular values = column norms, sorted descending (stable by index)
  for (int c = gwarp; c < np; c += nwarps) {
    double a = 0.0;
    for (int i = lane; i < np; i += 32) a = fma(W[(int64_t)c * np + i], W[(int64_t)c * np + i], a);
    a = warp_sum(a);
    if (lane == 0) cn[c] = sqrt(a);
  }
  grid.sync();
  for (int c = gwarp; c < n; c += nwarps) {
    const double sc = cn[c];
    int rank = 0;
    for (int d = lane; d < np; d += 32) {
      const double sd = cn[d];
      rank += (sd > sc || (sd == sc && d < c)) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (rank >= n) continue;
    if (lane == 0) S[rank] = sc;
    const double inv = sc > 0.0 ? 1.0 / sc : 0.0;
    for (int i = lane; i < n; i += 32) {
      U[(int64_t)i * ldu + rank] = W[(int64_t)c * np + i] * inv;
      if (Vout) Vout[(int64_t)i * ldv + rank] = Vm[(int64_t)c * np + i];
    }
  }
}

// ------------------------------------------ 32 < n <= 256, block rounds ----
// The Rayleigh-Ritz cores of the ID range finder (b = 40 ... 256).  The scalar
// kernels above pay one (grid) barrier and an L2 round trip per column-pair
// round: 255 rounds x ~6 sweeps at n = 256, 8 us each (12.5 ms per core, the
// largest item of a cfg3 power_id).  Here the columns are cut into 16-wide
// blocks and every OUTER round gives each CTA one block pair (round-robin over
// the blocks: nb - 1 outer rounds per sweep, one grid barrier each); the CTA
// holds the pair's 32 columns of W stacked on the same columns of V in shared
// memory (2 np rows, 128 KB at n = 256) and rotates all 16 x 16 cross pairs in
// 16 inner rounds of 16 disjoint pairs (one warp per pair, block barriers
// only); the pairs inside a block are rotated in the first outer round of the
// sweep, so a sweep visits every pair exactly once.  Rotations, thresholds,
// the quadratic-convergence stop and the sorted outputs are those of the
// scalar kernels.
constexpr int kJbW = 16;           // block width
constexpr int kJbThreads = 512;    // one warp per pair of the 32 resident columns

template <int RPL>  // rows of W per lane (np = 32 RPL)
__device__ __forceinline__ void jb_rotate(double* __restrict__ cp, double* __restrict__ cq, int lane, double negl,
                                          int* rot) {
  double x[2 * RPL], y[2 * RPL];
#pragma unroll
  for (int j = 0; j < RPL; ++j) {
    x[j] = cp[lane + 32 * j];
    y[j] = cq[lane + 32 * j];
  }
  double a = 0.0, b = 0.0, g = 0.0;
#pragma unroll
  for (int j = 0; j < RPL; ++j) {
    a = fma(x[j], x[j], a);
    b = fma(y[j], y[j], b);
    g = fma(x[j], y[j], g);
  }
  a = warp_sum(a);
  b = warp_sum(b);
  g = warp_sum(g);
  // thresholds on squares (no square roots) unless the product could overflow;
  // the rotation from two dependent MUFU rsqrt stages (the jacobi32 forms: the
  // IEEE sqrt / division sequences of the scalar kernels put ~3000 cycles of
  // dependent FP64 instructions on every round's critical path)
  const double ab = a * b;
  const bool big = !(ab < 1e300);
  if (!(g != 0.0 && fmin(a, b) > negl &&
        (big ? fabs(g) > kJacTol * sqrt(a) * sqrt(b) : g * g > (kJacTol * kJacTol) * ab)))
    return;
  const double d = b - a, h = 2.0 * g;
  const double ad = fabs(d), ah = fabs(h);
  double cs, sn;
  bool wide;  // large-angle rotation (see kJacFloor)
  if (ad < 1e140 && ah < 1e140 && (ad > 1e-140 || ah > 1e-140)) {
    const double s2 = fma(d, d, h * h);
    const double rh = fast_rsqrt(s2);
    const double u = fma(0.5 * ad, rh, 0.5);
    const double w = fast_rsqrt(u);
    cs = u * w;
    sn = (copysign(0.5, d) * h) * (rh * w);
    wide = h * h > kJacSin2 * s2;
  } else {
    const double t = copysign(1.0, d) * h / (ad + hypot(d, h));
    cs = rsqrt(fma(t, t, 1.0));
    sn = cs * t;
    wide = fabs(t) > 5e-5;
  }
#pragma unroll
  for (int j = RPL; j < 2 * RPL; ++j) {  // the V half
    x[j] = cp[lane + 32 * j];
    y[j] = cq[lane + 32 * j];
  }
#pragma unroll
  for (int j = 0; j < 2 * RPL; ++j) {
    cp[lane + 32 * j] = fma(-sn, y[j], cs * x[j]);
    cq[lane + 32 * j] = fma(sn, x[j], cs * y[j]);
  }
  // a rotation of relative size above kJacQuad keeps the sweeps going
  if (lane == 0) {
    int fl = wide ? kJfWide : 0;
    if (big ? fabs(g) > kJacQuad * sqrt(a) * sqrt(b) : g * g > (kJacQuad * kJacQuad) * ab) fl |= kJfQuad;
    if (big ? fabs(g) > kJacFloor * sqrt(a) * sqrt(b) : g * g > (kJacFloor * kJacFloor) * ab) fl |= kJfFloor;
    if (fl & ~*(volatile int*)rot) atomicOr(rot, fl);
  }
}

template <int RPL>
__global__ void __launch_bounds__(kJbThreads)
jacobi_blk_kernel(int n, const double* __restrict__ M, int64_t ldm, bool trans, double* __restrict__ U,
                  int64_t ldu, double* __restrict__ S, double* __restrict__ Vout, int64_t ldv,
                  double* __restrict__ W, double* __restrict__ Vm, double* __restrict__ cn, int* rot,
                  unsigned long long* relmax) {
  constexpr int np = 32 * RPL;
  constexpr int nb = np / kJbW;  // even
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double cols[];  // 32 columns x [W (np) | V (np)]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + tid;
  const int64_t gthr = (int64_t)gridDim.x * blockDim.x;
  const int gwarp = (int)(gtid >> 5), nwarps = (int)(gthr >> 5);
  for (int64_t e = gtid; e < (int64_t)np * np; e += gthr) {
    const int c = (int)(e / np), i = (int)(e % np);
    W[e] = (i < n && c < n) ? (trans ? M[(int64_t)c * ldm + i] : M[(int64_t)i * ldm + c]) : 0.0;
    Vm[e] = (i == c) ? 1.0 : 0.0;
  }
  if (gtid < 2) {
    rot[gtid] = 0;
    relmax[gtid] = 0ull;
  }
  grid.sync();
  for (int c = gwarp; c < np; c += nwarps) {
    double a = 0.0;
    for (int i = lane; i < np; i += 32) a = fma(W[(int64_t)c * np + i], W[(int64_t)c * np + i], a);
    a = warp_sum(a);
    if (lane == 0) cn[c] = a;
  }
  grid.sync();
  double fro = 0.0;
  for (int c = 0; c < np; ++c) fro += cn[c];
  const double negl = 1e-30 * fro;
  for (int sweep = 0; sweep < kJacMaxSweeps; ++sweep) {
    int* rt = &rot[sweep & 1];  // set by a rotation above kJacQuad in relative size
    for (int round = 0; round < nb - 1; ++round) {
      if (round == 1 && gtid == 0) rot[(sweep + 1) & 1] = 0;  // nobody reads the other parity until this sweep ends
      int bi, bj;
      rr_pair(nb, round, blockIdx.x, bi, bj);
      // stage the pair's columns: W half, then V half
      for (int e = tid; e < 32 * (np / 2); e += kJbThreads) {  // double2 units
        const int c = e / (np / 2), i2 = e % (np / 2);
        const int gc = (c < kJbW ? bi * kJbW + c : bj * kJbW + (c - kJbW));
        reinterpret_cast<double2*>(cols + (size_t)c * 2 * np)[i2] =
            reinterpret_cast<const double2*>(W + (int64_t)gc * np)[i2];
        reinterpret_cast<double2*>(cols + (size_t)c * 2 * np + np)[i2] =
            reinterpret_cast<const double2*>(Vm + (int64_t)gc * np)[i2];
      }
      __syncthreads();
      if (round == 0) {
        // pairs inside each block: warps 0-7 block bi, 8-15 block bj
        const int half = warp >> 3, k = warp & 7;
        for (int r = 0; r < kJbW - 1; ++r) {
          int p, q;
          rr_pair(kJbW, r, k, p, q);
          jb_rotate<RPL>(cols + (size_t)(half * kJbW + p) * 2 * np, cols + (size_t)(half * kJbW + q) * 2 * np, lane,
                         negl, rt);
          __syncthreads();
        }
      }
      for (int r = 0; r < kJbW; ++r) {
        const int p = warp, q = kJbW + ((warp + r) & (kJbW - 1));
        jb_rotate<RPL>(cols + (size_t)p * 2 * np, cols + (size_t)q * 2 * np, lane, negl, rt);
        __syncthreads();
      }
      for (int e = tid; e < 32 * (np / 2); e += kJbThreads) {
        const int c = e / (np / 2), i2 = e % (np / 2);
        const int gc = (c < kJbW ? bi * kJbW + c : bj * kJbW + (c - kJbW));
        reinterpret_cast<double2*>(W + (int64_t)gc * np)[i2] =
            reinterpret_cast<const double2*>(cols + (size_t)c * 2 * np)[i2];
        reinterpret_cast<double2*>(Vm + (int64_t)gc * np)[i2] =
            reinterpret_cast<const double2*>(cols + (size_t)c * 2 * np + np)[i2];
      }
      grid.sync();
    }
    // the stopping rule above
    if (!jac_continue(*(volatile int*)rt)) {
#ifdef SPB_JACOBI_TRACE
      if (gtid == 0) printf("jacobi_blk n=%d np=%d sweeps=%d\n", n, np, sweep + 1);
#endif
      break;
    }
  }
  // singular values = column norms, sorted descending (stable by index)
  for (int c = gwarp; c < np; c += nwarps) {
    double a = 0.0;
    for (int i = lane; i < np; i += 32) a = fma(W[(int64_t)c * np + i], W[(int64_t)c * np + i], a);
    a = warp_sum(a);
    if (lane == 0) cn[c] = sqrt(a);
  }
  grid.sync();
  for (int c = gwarp; c < n; c += nwarps) {
    const double sc = cn[c];
    int rank = 0;
    for (int d = lane; d < np; d += 32) {
      const double sd = cn[d];
      rank += (sd > sc || (sd == sc && d < c)) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (rank >= n) continue;
    if (lane == 0) S[rank] = sc;
    const double inv = sc > 0.0 ? 1.0 / sc : 0.0;
    for (int i = lane; i < n; i += 32) {
      U[(int64_t)i * ldu + rank] = W[(int64_t)c * np + i] * inv;
      if (Vout) Vout[(int64_t)i * ldv + rank] = Vm[(int64_t)c * np + i];
    }
  }
}

template <int RPL>
static int jacobi_blk_launch(int n, const double* M, int64_t ldm, bool trans, double* U, int64_t ldu, double* S,
                             double* V, int64_t ldv, cudaStream_t s) {
  constexpr int np = 32 * RPL;
  Arena gar(s);
  double* gW = gar.alloc<double>((size_t)np * np);
  double* gV = gar.alloc<double>((size_t)np * np);
  double* cn = gar.alloc<double>((size_t)np);
  int* rot = gar.alloc<int>(2);
  unsigned long long* relmax = gar.alloc<unsigned long long>(2);
  if (!gW || !gV || !cn || !rot || !relmax) {
    set_error("jacobi workspace allocation failed");
    return SP_ECUDA;
  }
  const size_t smem = (size_t)32 * 2 * np * sizeof(double);
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    SPB_CUDA(cudaFuncSetAttribute(jacobi_blk_kernel<RPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_dev = dev;
  }
  const int grid = np / kJbW / 2;
  void* args[] = {&n, &M, &ldm, &trans, &U, &ldu, &S, &V, &ldv, &gW, &gV, &cn, &rot, &relmax};
  SPB_CUDA(cudaLaunchCooperativeKernel((const void*)jacobi_blk_kernel<RPL>, dim3(grid), dim3(kJbThreads), args, smem, s));
  count_launch();
  return SP_OK;
}

static int jacobi_blk(int n, const double* M, int64_t ldm, bool trans, double* U, int64_t ldu, double* S, double* V,
                      int64_t ldv, cudaStream_t s) {
  switch ((n + 31) / 32) {
    case 2: return jacobi_blk_launch<2>(n, M, ldm, trans, U, ldu, S, V, ldv, s);
    case 3: return jacobi_blk_launch<3>(n, M, ldm, trans, U, ldu, S, V, ldv, s);
    case 4: return jacobi_blk_launch<4>(n, M, ldm, trans, U, ldu, S, V, ldv, s);
    case 5: return jacobi_blk_launch<5>(n, M, ldm, trans, U, ldu, S, V, ldv, s);
    case 6: return jacobi_blk_launch<6>(n, M, ldm, trans, U, ldu, S, V, ldv, s);
    case 7: return jacobi_blk_launch<7>(n, M, ldm, trans, U, ldu, S, V, ldv, s);
    default: return jacobi_blk_launch<8>(n, M, ldm, trans, U, ldu, S, V, ldv, s);
  }
}

// batch independent n x n SVDs (n <= 32), core b at M + b bsM (its U, S, V
// likewise): the pair solves of the block Jacobi (bjacobi.cu)
int jacobi32_batched(int n, int batch, const double* M, int64_t ldm, int64_t bsM, double* U, int64_t ldu,
                     int64_t bsU, double* S, int64_t bsS, double* V, int64_t ldv, int64_t bsV, cudaStream_t s) {
  SPB_REQUIRE(n >= 1 && n <= 32 && batch >= 1, "jacobi32_batched: 1 <= n <= 32");
  jacobi32_kernel<kJ32Warps, 8><<<batch, kJ32Warps * 32, 0, s>>>(n, M, ldm, U, ldu, S, V, ldv, false, bsM, bsU, bsS,
                                                                  bsV);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

int jacobi_svd(int64_t n, const double* M, int64_t ldm, double* U, int64_t ldu, double* S,
               double* V, int64_t ldv, cudaStream_t s) {
  return jacobi_svd_tr(n, M, ldm, false, U, ldu, S, V, ldv, s);
}

// SVD of M (trans = false) or of M^T (trans = true, n <= 32 reads M
// transposed in place; larger n transposes into scratch first)
int jacobi_svd_tr(int64_t n, const double* M, int64_t ldm, bool trans, double* U, int64_t ldu, double* S,
                  double* V, int64_t ldv, cudaStream_t s) {
  SPB_REQUIRE(n >= 1 && n <= 50000, "Jacobi SVD supports 1 <= n <= 50000");
  if (n <= 8) {
    SPB_CUDA(launch_pdl((jacobi32_kernel<1, 8>), dim3(1), dim3(32), 0, s, (int)n, M, ldm, U, ldu, S, V, ldv, trans,
                        (int64_t)0, (int64_t)0, (int64_t)0, (int64_t)0));
    count_launch();
    SPB_CHECK_LAUNCH();
    return SP_OK;
  }
  if (n <= 32) {
    SPB_CUDA(launch_pdl((jacobi32_kernel<kJ32Warps, 8>), dim3(1), dim3(kJ32Warps * 32), 0, s, (int)n, M, ldm, U, ldu, S,
                        V, ldv, trans, (int64_t)0, (int64_t)0, (int64_t)0, (int64_t)0));
    count_launch();
    SPB_CHECK_LAUNCH();
    return SP_OK;
  }
  // SPB_JACOBI_SCALAR=1: the scalar kernels for every n > 32 (comparison)
  static const bool scalar_only = getenv("SPB_JACOBI_SCALAR") != nullptr;
  if (n <= 256 && !scalar_only) return jacobi_blk((int)n, M, ldm, trans, U, ldu, S, V, ldv, s);
  Arena vscratch(s);
  if (trans) {
    double* Mt = vscratch.alloc<double>((size_t)n * n);
    if (!Mt) {
      set_error("jacobi workspace allocation failed");
      return SP_ECUDA;
    }
    SPB_TRY(transpose(n, n, M, ldm, Mt, n, s));
    M = Mt;
    ldm = n;
  }
  if (V == nullptr) {  // the multi-warp kernel always accumulates V
    V = vscratch.alloc<double>((size_t)n * n);
    ldv = n;
    if (!V) {
      set_error("jacobi workspace allocation failed");
      return SP_ECUDA;
    }
  }
  const int np = std::max<int>(2, (int)(n + (n & 1)));
  const int threads = std::min(1024, std::max(64, 32 * (np / 2)));
  const size_t smem = (size_t)2 * np * np * sizeof(double);
  const bool use_smem = smem <= 200 * 1024;
  if (!use_smem) {
    // cooperative grid: one warp per column pair, W / V in global memory
    Arena gar(s);
    double* gW = gar.alloc<double>((size_t)np * np);
    double* gV = gar.alloc<double>((size_t)np * np);
    double* cn = gar.alloc<double>((size_t)np);
    int* rot = gar.alloc<int>(2);
    unsigned long long* relmax = gar.alloc<unsigned long long>(2);
    if (!gW || !gV || !cn || !rot || !relmax) {
      set_error("jacobi workspace allocation failed");
      return SP_ECUDA;
    }
    const int warps = np / 2;
    int grid = ceil_div(warps * 32, kJgThreads);
    const size_t act_smem = (size_t)np * sizeof(int);
    if (act_smem > 48 * 1024)
      SPB_CUDA(cudaFuncSetAttribute(jacobi_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)act_smem));
    int per_sm = 0;
    SPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_grid_kernel, kJgThreads, act_smem));
    grid = std::max(1, std::min(grid, per_sm * kNumSMs));
    int n_i = (int)n, np_i = np;
    bool tr = false;  // M was transposed into scratch above when trans
    void* args[] = {&n_i, &np_i, &M, &ldm, &tr, &U, &ldu, &S, &V, &ldv, &gW, &gV, &cn, &rot, &relmax};
    SPB_CUDA(cudaLaunchCooperativeKernel((const void*)jacobi_grid_kernel, dim3(grid), dim3(kJgThreads), args, act_smem,
                                         s));
    count_launch();
    return SP_OK;
  }
  Arena ar(s);
  double *gW = nullptr, *gV = nullptr;
  if (!use_smem) {
    gW = ar.alloc<double>((size_t)np * np);
    gV = ar.alloc<double>((size_t)np * np);
    if (!gW || !gV) {
      set_error("jacobi workspace allocation failed");
      return SP_ECUDA;
    }
  } else {
    SPB_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  jacobi_kernel<<<1, threads, use_smem ? smem : 0, s>>>((int)n, np, M, ldm, U, ldu, S, V, ldv, gW, gV,
                                                        use_smem);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

}  // namespace spb
