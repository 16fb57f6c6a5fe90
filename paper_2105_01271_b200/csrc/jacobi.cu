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
#include "common.cuh"
#include "launch_count.cuh"

namespace spb {

constexpr int kJacMaxSweeps = 40;
constexpr double kJacTol = 1e-15;

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
  for (int sweep = 0; sweep < kJacMaxSweeps && na >= 2; ++sweep) {
    if (tid == 0) rot_count = 0;
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
          if (lane == 0) atomicAdd(&rot_count, 1);
        }
      }
      __syncthreads();
    }
    if (rot_count == 0) break;
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

int jacobi_svd(int64_t n, const double* M, int64_t ldm, double* U, int64_t ldu, double* S,
               double* V, int64_t ldv, cudaStream_t s) {
  SPB_REQUIRE(n >= 1 && n <= 256, "Jacobi SVD supports 1 <= n <= 256");
  const int np = std::max<int>(2, (int)(n + (n & 1)));
  const int threads = std::min(1024, std::max(64, 32 * (np / 2)));
  const size_t smem = (size_t)2 * np * np * sizeof(double);
  const bool use_smem = smem <= 200 * 1024;
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
