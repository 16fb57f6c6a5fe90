// Block one-sided Jacobi SVD for wide cores (many active columns).
//
// The one-sided (Hestenes) Jacobi of jacobi.cu rotates one column pair per
// warp and crosses a cooperative-grid barrier every round: n - 1 rounds per
// sweep, each touching all of W and V -- ~90 us a round once W and V leave
// the L2 (n = 4096: ~3.5 s).  Here the n columns are cut into 16-column
// blocks and every round rotates nb / 2 block PAIRS at once (nb - 1 rounds per
// sweep, 16x fewer): for each pair X_p = [W_I W_J] (N x 32)
//
//   1. R_p: Cholesky of the double-double Gram X_p^T X_p (one CTA per pair;
//      ~106-bit Gram, so R_p carries the Householder backward error
//      eps ||X_p||, as in ddgram.cu; pivots below 1e-29 tr(G) give zero rows);
//   2. the one-sided Jacobi SVD of R_p = U_p S_p V_p^T (jacobi32, batched);
//   3. X_p <- X_p V_p and the accumulated rotations V[:, pair] <- V[:, pair] V_p
//      (one thread per row, V_p in shared memory).
//
// X_p V_p = Q_p U_p S_p has orthogonal columns: the pair is exactly
// orthogonalised every round (a block rotation), and a sweep visits every
// block pair once (circle schedule).  Convergence: the largest relative
// cross-block Gram entry |g_ij| / sqrt(g_ii g_jj) of a sweep; a sweep below
// 1e-11 is the last, below 1e-15 nothing rotates.
// Used by the size-general thin_svd when more than 512 columns are active
// (the sketch cores of cfg3 / cfg5 in their noise bulk, and full-rank drop-in
// inputs); the final column norms are the singular values.
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

// batched jacobi32 (jacobi.cu): SVD of M_b (n x n, ld ldm) for b < batch
int jacobi32_batched(int n, int batch, const double* M, int64_t ldm, int64_t bsM, double* U, int64_t ldu,
                     int64_t bsU, double* S, int64_t bsS, double* V, int64_t ldv, int64_t bsV, cudaStream_t s);

namespace {

constexpr int kBw = 16;          // block width
constexpr int kBp = 2 * kBw;     // pair width
constexpr int kBpEnt = kBp * (kBp + 1) / 2;
constexpr int kBgThreads = 288;  // 2 Gram entries per thread
constexpr int kBgTile = 64;      // rows staged per step
constexpr double kBgFloor = 1e-29;

struct bdd {
  double hi, lo;
};
__device__ __forceinline__ bdd b_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ bdd b_quick(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ bdd b_add(bdd a, bdd b) {
  bdd s = b_two_sum(a.hi, b.hi);
  const bdd t = b_two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = b_quick(s.hi, s.lo);
  s.lo += t.lo;
  return b_quick(s.hi, s.lo);
}
__device__ __forceinline__ bdd b_mul(bdd a, bdd b) {
  const double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e = fma(a.hi, b.lo, e);
  e = fma(a.lo, b.hi, e);
  return b_quick(p, e);
}

__device__ __forceinline__ void b_entry(int e, int& i, int& j) {
  if (e >= kBpEnt) {
    i = j = 0;
    return;
  }
  int r = 0, base = 0;
  while (e >= base + (kBp - r)) {
    base += kBp - r;
    ++r;
  }
  i = r;
  j = r + (e - base);
}

// circle schedule over nbp (even) blocks: pair k of round r -> (p, q), p < q
__device__ __forceinline__ void b_pair(int nbp, int round, int k, int& p, int& q) {
  const int n1 = nbp - 1;
  if (k == 0) {
    p = 0;
    q = 1 + (round % n1);
  } else {
    p = 1 + ((round + k) % n1);
    q = 1 + ((round - k + n1) % n1);
  }
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

constexpr int kBgRows = 512;     // rows per Gram-partial CTA

// Gram partials: CTA (pair, split) accumulates the dd Gram of its row range
// of the pair's 32 columns of W (column-major, column c at W + c ldw; blocks
// >= nb are empty padding) -> part[(pair * nsplit + split) * kBpEnt + e], e
// the row-major upper-triangle index; two entries per thread (a 4 x 4
// register-blocked variant needed 150 registers, one CTA per SM, and ran
// 1.8x slower).
__global__ void __launch_bounds__(kBgThreads)
bj_gram_part_kernel(int64_t N, int nb, int nbp, int round, int nsplit, const double* __restrict__ W, int64_t ldw,
                    double2* __restrict__ part) {
  __shared__ __align__(16) double xs[kBp][kBgTile + 1];
  int bp, bq;
  b_pair(nbp, round, blockIdx.x, bp, bq);
  if (bq >= nb) return;
  const int t = threadIdx.x;
  int ei[2], ej[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) b_entry(2 * t + u, ei[u], ej[u]);
  double hi[2] = {0.0, 0.0}, lo[2] = {0.0, 0.0};
  const int64_t offp = (int64_t)bp * kBw, offq = (int64_t)bq * kBw;
  const int64_t r0 = (int64_t)blockIdx.y * kBgRows, r1 = imin64(N, r0 + kBgRows);
  for (int64_t c0 = r0; c0 < r1; c0 += kBgTile) {
    const int nr = (int)imin64(kBgTile, r1 - c0);
    for (int e = t; e < kBgTile * kBp; e += kBgThreads) {
      const int cc = e / kBgTile, rr = e % kBgTile;  // consecutive threads: consecutive rows (coalesced)
      const int64_t col = cc < kBw ? offp + cc : offq + (cc - kBw);
      xs[cc][rr] = rr < nr ? W[col * ldw + c0 + rr] : 0.0;
    }
    __syncthreads();
    if (2 * t < kBpEnt) {
#pragma unroll 4
      for (int rr = 0; rr < kBgTile; ++rr) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const double xi = xs[ei[u]][rr], xj = xs[ej[u]][rr];
          const double p = xi * xj;
          const double pe = fma(xi, xj, -p);
          const double sm = hi[u] + p;
          const double bb = sm - hi[u];
          lo[u] += ((hi[u] - (sm - bb)) + (p - bb)) + pe;
          hi[u] = sm;
        }
      }
    }
    __syncthreads();
  }
  if (2 * t < kBpEnt) {
    double2* dst = part + ((int64_t)blockIdx.x * nsplit + blockIdx.y) * kBpEnt;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const bdd a = b_quick(hi[u], lo[u]);
      dst[2 * t + u] = make_double2(a.hi, a.lo);
    }
  }
}

// one CTA per pair: the partials summed in split order (dd), the sweep
// statistic, and the dd Cholesky -> R_p (32 x 32 row-major, zeros below the
// diagonal; pivots below 1e-29 tr(G) give zero rows)
__global__ void __launch_bounds__(kBgThreads)
bj_chol_kernel(int nb, int nbp, int round, int nsplit, const double2* __restrict__ part, double* __restrict__ Rb,
               unsigned long long* relmax) {
  __shared__ bdd S[kBp][kBp + 1];
  __shared__ double piv_r[2];
  __shared__ bdd piv_d[2];
  int bp, bq;
  b_pair(nbp, round, blockIdx.x, bp, bq);
  double* R = Rb + (int64_t)blockIdx.x * kBp * kBp;
  const int t = threadIdx.x;
  if (bq >= nb) {  // a pair with the padding block: not rotated
    for (int e = t; e < kBp * kBp; e += blockDim.x) R[e] = 0.0;
    return;
  }
  int ei[2], ej[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) b_entry(2 * t + u, ei[u], ej[u]);
  if (2 * t < kBpEnt) {
    const double2* src = part + (int64_t)blockIdx.x * nsplit * kBpEnt;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      bdd a = {0.0, 0.0};
      for (int q = 0; q < nsplit; ++q) {
        const double2 v = src[(int64_t)q * kBpEnt + 2 * t + u];
        a = b_add(a, {v.x, v.y});
      }
      S[ei[u]][ej[u]] = a;
    }
  }
  __syncthreads();
  // sweep statistic: the largest relative cross-block entry
  {
    double mx = 0.0;
    if (2 * t < kBpEnt) {
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (ei[u] < kBw && ej[u] >= kBw) {
          const double gii = S[ei[u]][ei[u]].hi, gjj = S[ej[u]][ej[u]].hi;
          const double g = fabs(S[ei[u]][ej[u]].hi);
          if (gii > 0.0 && gjj > 0.0) mx = fmax(mx, g / (sqrt(gii) * sqrt(gjj)));
        }
    }
    mx = warp_max(mx);
    if ((t & 31) == 0 && mx > 0.0) atomicMax(relmax, (unsigned long long)__double_as_longlong(mx));
  }
  double tr = 0.0;
  for (int j = 0; j < kBp; ++j) tr += S[j][j].hi;
  const double floor_abs = kBgFloor * tr;
  const int gi = t >> 3, j0 = (t & 7) * 4;
  const bool ct = t < 256;
  auto pivot = [&](bdd d, int buf) {
    if (d.hi > floor_abs && d.hi < 1e300) {
      piv_r[buf] = 1.0 / sqrt(d.hi);
      const double q1 = 1.0 / d.hi;
      const double p = d.hi * q1;
      const double e = fma(d.hi, q1, -p);
      const double r = fma(-d.lo, q1, (1.0 - p) - e);
      piv_d[buf] = b_quick(q1, r * q1);
    } else {
      piv_r[buf] = 0.0;
      piv_d[buf] = {0.0, 0.0};
    }
  };
  if (t == 0) pivot(S[0][0], 0);
  __syncthreads();
  for (int j = 0; j < kBp; ++j) {
    const double rinv = piv_r[j & 1];
    const bdd inv2 = piv_d[j & 1];
    if (ct && gi == j) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = j0 + u;
        R[j * kBp + k] = k >= j ? S[j][k].hi * rinv : 0.0;
      }
    }
    if (ct && gi > j) {
      bdd rowj[4], mine[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        rowj[u] = S[j][j0 + u];
        mine[u] = S[gi][j0 + u];
      }
      if (inv2.hi != 0.0) {
        const bdd f = b_mul(S[j][gi], inv2);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bdd pr = b_mul(f, rowj[u]);
          mine[u] = b_add(mine[u], {-pr.hi, -pr.lo});
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = j0 + u;
          if (k >= gi) S[gi][k] = mine[u];
        }
      }
      if (gi == j + 1 && j0 <= gi && gi < j0 + 4) {
        bdd dnext = mine[0];
#pragma unroll
        for (int u = 1; u < 4; ++u)
          if (j0 + u == gi) dnext = mine[u];
        pivot(dnext, (j + 1) & 1);
      }
    }
    __syncthreads();
  }
}

// X_p <- X_p V_p for the pair's 32 columns of W (N rows, column-major, ld
// ldw) and of the rotation accumulator Va (nv rows, ld ldv); V_p (32 x 32
// row-major) in shared memory; one thread per row (coalesced column loads),
// the 32 outputs in registers.  No row loop: a loop lets the compiler hoist
// the 1024 loop-invariant V_p reads into registers and spill them.  Pairs
// with the padding block are left alone.
__global__ void __launch_bounds__(256)
bj_apply_kernel(int64_t N, int64_t nv, int nb, int nbp, int round, double* __restrict__ W, int64_t ldw,
                double* __restrict__ Va, int64_t ldv, const double* __restrict__ Vb) {
  __shared__ double vp[kBp][kBp];
  int bp, bq;
  b_pair(nbp, round, blockIdx.y, bp, bq);
  if (bq >= nb) return;
  const double* V = Vb + (int64_t)blockIdx.y * kBp * kBp;
  for (int e = threadIdx.x; e < kBp * kBp; e += blockDim.x) vp[e / kBp][e % kBp] = V[e];
  __syncthreads();
  const int64_t offp = (int64_t)bp * kBw, offq = (int64_t)bq * kBw;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N + nv) return;
  double* base = r < N ? W + r : Va + (r - N);
  const int64_t ld = r < N ? ldw : ldv;
  double* pp = base + offp * ld;
  double* pq = base + offq * ld;
  double y[kBp];
#pragma unroll
  for (int c = 0; c < kBp; ++c) y[c] = 0.0;
#pragma unroll
  for (int k = 0; k < kBp; ++k) {
    const double xk = k < kBw ? pp[k * ld] : pq[(k - kBw) * ld];
#pragma unroll
    for (int c = 0; c < kBp; ++c) y[c] = fma(xk, vp[k][c], y[c]);
  }
#pragma unroll
  for (int c = 0; c < kBw; ++c) {
    pp[c * ld] = y[c];
    pq[c * ld] = y[kBw + c];
  }
}

// column norms of W (N x npad, column-major) and, per column, whether the
// accumulated rotation there is a padding coordinate's unit vector (padding
// coordinates never mix with real ones: their columns are zero, outside every
// pair rotation's active set, and only move by the pair SVD's sorting); one
// warp per column
__global__ void bj_norms_kernel(int64_t N, int64_t npad, int64_t n, const double* __restrict__ W, int64_t ldw,
                                const double* __restrict__ Va, int64_t ldva, double* __restrict__ nrm,
                                int* __restrict__ pad) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= npad) return;
  double a = 0.0;
  for (int64_t r = lane; r < N; r += 32) a = fma(W[c * ldw + r], W[c * ldw + r], a);
  a = warp_sum(a);
  double p = 0.0;
  for (int64_t r = n + lane; r < npad; r += 32) p = fma(Va[c * ldva + r], Va[c * ldva + r], p);
  p = warp_sum(p);
  if (lane == 0) {
    nrm[c] = sqrt(a);
    pad[c] = p > 0.5 ? 1 : 0;
  }
}

// sorted output: S[rank] = nrm[c], U[:, rank] = W[:, c] / nrm[c],
// V[:, rank] = Va[:, c] (U, V row-major); rank by (real before padding,
// descending norm, index)
__global__ void bj_sort_out_kernel(int64_t N, int64_t n, const double* __restrict__ W, int64_t ldw,
                                   const double* __restrict__ Va, int64_t ldva, const double* __restrict__ nrm,
                                   const int* __restrict__ pad, double* __restrict__ U, int64_t ldu,
                                   double* __restrict__ S, double* __restrict__ V, int64_t ldv) {
  const int64_t c = blockIdx.x;
  __shared__ unsigned long long rk_s;
  if (threadIdx.x == 0) rk_s = 0;
  __syncthreads();
  const double sc = nrm[c];
  const int pc = pad[c];
  unsigned long long rk = 0;
  for (int64_t d = threadIdx.x; d < n; d += blockDim.x) {
    const double sd = nrm[d];
    const int pd = pad[d];
    rk += (pd < pc || (pd == pc && (sd > sc || (sd == sc && d < c)))) ? 1 : 0;
  }
  atomicAdd(&rk_s, rk);
  __syncthreads();
  const int64_t rank = (int64_t)rk_s;
  if (threadIdx.x == 0) S[rank] = sc;
  const double inv = sc > 0.0 ? 1.0 / sc : 0.0;
  for (int64_t r = threadIdx.x; r < N; r += blockDim.x) U[r * ldu + rank] = W[c * ldw + r] * inv;
  for (int64_t r = threadIdx.x; r < n; r += blockDim.x) V[r * ldv + rank] = Va[c * ldva + r];
}

// W (N x npad, column-major) = M (or M^T) zero-padded; Va = I (npad x npad)
__global__ void bj_init_kernel(int64_t N, int64_t n, int64_t npad, const double* __restrict__ M, int64_t ldm, bool trans,
                               double* __restrict__ W, double* __restrict__ Va) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t wtot = N * npad;
  if (e < wtot) {
    const int64_t c = e / N, r = e % N;
    W[e] = c < n ? (trans ? M[c * ldm + r] : M[r * ldm + c]) : 0.0;
  } else if (e < wtot + npad * npad) {
    const int64_t f = e - wtot, c = f / npad, r = f % npad;
    Va[f] = r == c ? 1.0 : 0.0;
  }
}

}  // namespace

// SVD of M (N x n, ld ldm; trans: M is given transposed, n x N) by block
// Jacobi: U (N x n, ld ldu; the normalised rotated columns, zero where S = 0),
// S (n, descending), V (n x n, ld ldv; the rotations).  Synchronises once per sweep.
int block_jacobi_svd(int64_t N, int64_t n, const double* M, int64_t ldm, bool trans, double* U, int64_t ldu,
                     double* S, double* V, int64_t ldv, cudaStream_t s) {
  SPB_REQUIRE(N >= 1 && n >= 2, "block_jacobi_svd: empty input");
  const int nb = ceil_div(n, kBw);
  const int nbp = nb + (nb & 1);  // even: a padding block completes the circle
  const int64_t npad = (int64_t)nbp * kBw;
  const int npairs = nbp / 2;
  Arena ar(s);
  SPB_ALLOC(ar, double, W, (size_t)N * npad);
  SPB_ALLOC(ar, double, Va, (size_t)npad * npad);
  SPB_ALLOC(ar, double, Rb, (size_t)npairs * kBp * kBp);
  SPB_ALLOC(ar, double, Ub, (size_t)npairs * kBp * kBp);
  SPB_ALLOC(ar, double, Sb, (size_t)npairs * kBp);
  SPB_ALLOC(ar, double, Vb, (size_t)npairs * kBp * kBp);
  SPB_ALLOC(ar, unsigned long long, relmax, 64);
  SPB_ALLOC(ar, double, nrm, (size_t)npad);
  const int nsplit = ceil_div(N, kBgRows);
  SPB_ALLOC(ar, double2, gpart, (size_t)npairs * nsplit * kBpEnt);
  const int64_t init_n = N * npad + npad * npad;
  bj_init_kernel<<<ceil_div(init_n, 256), 256, 0, s>>>(N, n, npad, M, ldm, trans, W, Va);
  count_launch();
  SPB_CHECK_LAUNCH();
  SPB_CUDA(cudaMemsetAsync(relmax, 0, 64 * sizeof(unsigned long long), s));
  const int apply_x = ceil_div(N + npad, 256);  // one row per thread
  constexpr int kMaxSweeps = 40;
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    unsigned long long* rm = relmax + (sweep % 64);
    for (int round = 0; round < nbp - 1; ++round) {
      bj_gram_part_kernel<<<dim3(npairs, nsplit), kBgThreads, 0, s>>>(N, nb, nbp, round, nsplit, W, N, gpart);
      bj_chol_kernel<<<npairs, kBgThreads, 0, s>>>(nb, nbp, round, nsplit, gpart, Rb, rm);
      SPB_TRY(jacobi32_batched(kBp, npairs, Rb, kBp, kBp * kBp, Ub, kBp, kBp * kBp, Sb, kBp, Vb, kBp, kBp * kBp, s));
      bj_apply_kernel<<<dim3(apply_x, npairs), 256, 0, s>>>(N, npad, nb, nbp, round, W, N, Va, npad, Vb);
      count_launch(3);
      SPB_CHECK_LAUNCH();
    }
    unsigned long long h = 0;
    SPB_TRY(read_small(&h, rm, sizeof(h), s));
    double mx = 0.0;
    std::memcpy(&mx, &h, sizeof(mx));
    // A sweep whose cross-block couplings were all below 1e-8 leaves ~1e-16 behind when
    // the singular values are separated (quadratic convergence), but inside a cluster of
    // equal singular values the block rotations are large-angle and the other couplings
    // are mixed, not squared: stop only once a sweep starts below 1e-11 (one more sweep on
    // separated spectra; U, V orthonormal to 1e-10 on flat ones).
    if (mx < 1e-11) break;
  }
  SPB_ALLOC(ar, int, padf, (size_t)npad);
  bj_norms_kernel<<<ceil_div(npad * 32, 256), 256, 0, s>>>(N, npad, n, W, N, Va, npad, nrm, padf);
  count_launch();
  SPB_CHECK_LAUNCH();
  // the padding coordinates sort last; write the first n ranks only
  Arena out(s);
  SPB_ALLOC(out, double, Uf, (size_t)N * npad);
  SPB_ALLOC(out, double, Sf, (size_t)npad);
  SPB_ALLOC(out, double, Vf, (size_t)npad * npad);
  bj_sort_out_kernel<<<(unsigned)npad, 256, 0, s>>>(N, npad, W, N, Va, npad, nrm, padf, Uf, npad, Sf, Vf, npad);
  count_launch();
  SPB_CHECK_LAUNCH();
  SPB_TRY(copy2d(N, n, Uf, npad, U, ldu, s));
  SPB_CUDA(cudaMemcpyAsync(S, Sf, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  SPB_TRY(copy2d(n, n, Vf, npad, V, ldv, s));
  return SP_OK;
}

}  // namespace spb
