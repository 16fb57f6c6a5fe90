// K7 across ranks: the greedy pivoted QR of the ID (src/kernels.py:97-142)
// on a candidate matrix whose ROWS are sharded.
//
// The ID selects rows of the enriched sketch E (m x n_c); E is column-sharded
// like C (rank i holds E_i = W C_i, m x n_ci), so every candidate (a row of E)
// is split across the ranks.  Each step of the reference loop becomes local
// partial sums plus one allreduce per reduction -- no rank repeats another's
// work and nothing of E moves:
//
//   norms   ||w_j||^2 = sum_i ||w_j,i||^2           allreduce (m values)
//   select  argmax, lowest original index on ties   replicated (same sums)
//   reorth  delta = Q^T w_t = sum_i Q_i^T w_t,i     allreduce (t values)
//   pivot   ||v||^2   = sum_i ||v_i||^2             allreduce (1 value)
//   coefs   v . w_j   = sum_i v_i . w_j,i           allreduce (m values)
//   update  w_j,i -= coef_j v_i (local), next norms
//
// R (k x m) and the pivot order come out identical on every rank, so the
// interpolation coefficients R1^-1 R2 and P are replicated without further
// exchange.  The partial sums of each rank are reduced in a fixed order, and
// the allreduce result is the same on every rank, so the selection is
// deterministic.  The caller (sharded.py) owns the allreduces; these entry
// points are the per-rank device work between them.
#include <cmath>

#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

constexpr int kPdThreads = 256;
constexpr int kPdMaxK = 1024;

__device__ __forceinline__ double pd_block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double acc = 0.0;
#pragma unroll
  for (int w = 0; w < kPdThreads / 32; ++w) acc += red[w];
  return acc;
}

// WK = E_i (candidate j = row j, length len), perm = iota, pn2[j] = ||w_j,i||^2
__global__ void pd_init_kernel(int64_t m, int64_t len, const double* __restrict__ E, int64_t lde,
                               double* __restrict__ WK, int64_t* __restrict__ perm, double* __restrict__ pn2) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= m) return;
  double a = 0.0;
  for (int64_t x = lane; x < len; x += 32) {
    const double v = E[j * lde + x];
    WK[j * len + x] = v;
    a = fma(v, v, a);
  }
  a = warp_sum(a);
  if (lane == 0) {
    pn2[j] = a;
    perm[j] = j;
  }
}

struct PdBest {
  double nrm;
  int64_t perm;
  int64_t j;
};

__device__ __forceinline__ bool pd_better(const PdBest& a, const PdBest& b) {
  return a.nrm > b.nrm || (a.nrm == b.nrm && a.perm < b.perm);
}

// norms from the allreduced squares; argmax over j >= t (lowest original
// index on exact ties); swap the replicated state (perm, R columns) and the
// local candidate rows; delta_i[s] = q_s,i . w_t,i (s < t, local rows)
__global__ void __launch_bounds__(1024)
pd_select_kernel(int t, int k, int64_t m, int64_t len, const double* __restrict__ n2, int64_t* perm, double* R,
                 int64_t ldr, double* __restrict__ WK, const double* __restrict__ Qt, double* __restrict__ delta,
                 int64_t* jsel) {
  __shared__ PdBest bests[32];
  __shared__ int64_t js_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  PdBest b{-1.0, INT64_MAX, -1};
  for (int64_t j = t + tid; j < m; j += blockDim.x) {
    PdBest c{sqrt(n2[j]), perm[j], j};
    if (pd_better(c, b)) b = c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    PdBest c{__shfl_xor_sync(0xffffffffu, b.nrm, o), __shfl_xor_sync(0xffffffffu, b.perm, o),
             __shfl_xor_sync(0xffffffffu, b.j, o)};
    if (pd_better(c, b)) b = c;
  }
  if (lane == 0) bests[warp] = b;
  __syncthreads();
  if (tid == 0) {
    PdBest bb = bests[0];
    for (int w = 1; w < nw; ++w)
      if (pd_better(bests[w], bb)) bb = bests[w];
    js_s = bb.j;
    *jsel = bb.j;
  }
  __syncthreads();
  const int64_t js = js_s;
  if (js != t) {
    for (int s = tid; s < k; s += blockDim.x) {
      const double a = R[(int64_t)s * ldr + t];
      R[(int64_t)s * ldr + t] = R[(int64_t)s * ldr + js];
      R[(int64_t)s * ldr + js] = a;
    }
    for (int64_t x = tid; x < len; x += blockDim.x) {
      const double a = WK[(int64_t)t * len + x];
      WK[(int64_t)t * len + x] = WK[js * len + x];
      WK[js * len + x] = a;
    }
    if (tid == 0) {
      const int64_t p = perm[t];
      perm[t] = perm[js];
      perm[js] = p;
    }
  }
  __syncthreads();
  const double* wt = WK + (int64_t)t * len;
  for (int s = warp; s < t; s += nw) {
    double a = 0.0;
    for (int64_t x = lane; x < len; x += 32) a = fma(Qt[(int64_t)s * len + x], wt[x], a);
    a = warp_sum(a);
    if (lane == 0) delta[s] = a;
  }
}

// R[s][t] += delta[s] (allreduced); v_i = w_t,i - sum_s delta_s q_s,i into Qt
// row t; part2[0] = ||v_i||^2 (one CTA, fixed order)
__global__ void __launch_bounds__(kPdThreads)
pd_orth_kernel(int t, int64_t len, const double* __restrict__ delta, double* __restrict__ R, int64_t ldr,
               const double* __restrict__ WK, double* __restrict__ Qt, double* __restrict__ part2) {
  __shared__ double red[kPdThreads / 32];
  __shared__ double ds[kPdMaxK];
  for (int s = threadIdx.x; s < t; s += kPdThreads) {
    ds[s] = delta[s];
    R[(int64_t)s * ldr + t] += delta[s];
  }
  __syncthreads();
  const double* wt = WK + (int64_t)t * len;
  double* v = Qt + (int64_t)t * len;
  double p = 0.0;
  for (int64_t x = threadIdx.x; x < len; x += kPdThreads) {
    double acc = 0.0;
    for (int s = 0; s < t; ++s) acc = fma(Qt[(int64_t)s * len + x], ds[s], acc);
    const double vv = wt[x] - acc;
    v[x] = vv;
    p = fma(vv, vv, p);
  }
  p = pd_block_sum(p, red);
  if (threadIdx.x == 0) part2[0] = p;
}

// pn = sqrt(allreduced ||v||^2) -> R[t][t]; v_i /= pn; coef_i[j] = v_i . w_j,i
// (j > t; warp per candidate).  A zero pivot raises *status (the sharded
// driver reports it; the reference's deterministic filler needs the whole
// candidate and is left to the single-GPU path).
__global__ void pd_coef_kernel(int t, int64_t m, int64_t len, const double* __restrict__ p2, double* __restrict__ R,
                               int64_t ldr, const double* __restrict__ WK, double* __restrict__ Qt,
                               double* __restrict__ coef, int* status) {
  const double pn = sqrt(p2[0]);
  const int64_t j = t + 1 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    R[(int64_t)t * ldr + t] = pn;
    if (pn == 0.0) *status = SP_ENUMERICAL;
  }
  if (j >= m || pn == 0.0) return;
  const double* v = Qt + (int64_t)t * len;
  const double* w = WK + j * len;
  double a = 0.0;
  for (int64_t x = lane; x < len; x += 32) a = fma(v[x] / pn, w[x], a);
  a = warp_sum(a);
  if (lane == 0) coef[j] = a;
}

__global__ void pd_normalise_kernel(int t, int64_t len, const double* __restrict__ p2, double* __restrict__ Qt) {
  const double pn = sqrt(p2[0]);
  if (pn == 0.0) return;
  double* v = Qt + (int64_t)t * len;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < len; x += (int64_t)gridDim.x * blockDim.x)
    v[x] = v[x] / pn;
}

// R[t][j] = coef_j (allreduced); w_j,i -= coef_j v_i; pn2[j] = ||w_j,i||^2
__global__ void pd_update_kernel(int t, int64_t m, int64_t len, const double* __restrict__ coef, double* __restrict__ R,
                                 int64_t ldr, double* __restrict__ WK, const double* __restrict__ Qt,
                                 double* __restrict__ pn2) {
  const int64_t j = t + 1 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= m) return;
  const double c = coef[j];
  const double* v = Qt + (int64_t)t * len;
  double* w = WK + j * len;
  double a = 0.0;
  for (int64_t x = lane; x < len; x += 32) {
    const double nv = fma(-c, v[x], w[x]);
    w[x] = nv;
    a = fma(nv, nv, a);
  }
  a = warp_sum(a);
  if (lane == 0) {
    R[(int64_t)t * ldr + j] = c;
    pn2[j] = a;
  }
}

// ------------------------------------------------------------- entries ----
int pqd_begin(int64_t m, int64_t len, int k, const double* E, int64_t lde, double* WK, int64_t* perm, double* R,
              int64_t ldr, double* pn2, cudaStream_t s) {
  SPB_REQUIRE(k >= 1 && k <= kPdMaxK && k <= m, "sharded pivoted QR: need 1 <= k <= min(m, 1024)");
  SPB_CUDA(cudaMemset2DAsync(R, ldr * sizeof(double), 0, m * sizeof(double), k, s));
  pd_init_kernel<<<ceil_div(m * 32, 256), 256, 0, s>>>(m, len, E, lde, WK, perm, pn2);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

int pqd_select(int t, int k, int64_t m, int64_t len, const double* n2, int64_t* perm, double* R, int64_t ldr,
               double* WK, const double* Qt, double* delta, int64_t* jsel, cudaStream_t s) {
  pd_select_kernel<<<1, 1024, 0, s>>>(t, k, m, len, n2, perm, R, ldr, WK, Qt, delta, jsel);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

int pqd_orth(int t, int64_t len, const double* delta, double* R, int64_t ldr, const double* WK, double* Qt,
             double* part2, cudaStream_t s) {
  pd_orth_kernel<<<1, kPdThreads, 0, s>>>(t, len, delta, R, ldr, WK, Qt, part2);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

int pqd_coef(int t, int64_t m, int64_t len, const double* p2, double* R, int64_t ldr, const double* WK, double* Qt,
             double* coef, int* status, cudaStream_t s) {
  const int64_t trail = m - t - 1;
  pd_coef_kernel<<<std::max(1, ceil_div(std::max<int64_t>(trail, 1) * 32, 256)), 256, 0, s>>>(t, m, len, p2, R, ldr,
                                                                                             WK, Qt, coef, status);
  pd_normalise_kernel<<<std::max(1, std::min<int>(4 * kNumSMs, ceil_div(len, 256))), 256, 0, s>>>(t, len, p2, Qt);
  count_launch(2);
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

int pqd_update(int t, int64_t m, int64_t len, const double* coef, double* R, int64_t ldr, double* WK, const double* Qt,
               double* pn2, cudaStream_t s) {
  const int64_t trail = m - t - 1;
  if (trail <= 0) return SP_OK;
  pd_update_kernel<<<ceil_div(trail * 32, 256), 256, 0, s>>>(t, m, len, coef, R, ldr, WK, Qt, pn2);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

}  // namespace spb
