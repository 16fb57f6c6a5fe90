// K7: rank-k column-pivoted QR by modified Gram-Schmidt (src/kernels.py:97-142).
//
// The reference's pivot rule is reproduced exactly: at step t the residual
// norms of the columns t.. are compared, the largest wins, exact ties go to
// the smallest ORIGINAL column index (perm), the winner is swapped to t, one
// classical re-orthogonalisation against q_0..q_{t-1} is folded into R, a zero
// pivot is replaced by the first e_i with a large orthogonal residual, and the
// trailing columns get the rank-1 update.  The matrix is held transposed
// (each candidate column contiguous), so the norm of every updated column is
// recomputed in the same warp pass as its update -- the same quantity the
// reference recomputes from scratch at the start of the next step.
//
// Per step: one single-CTA "select" kernel (argmax, swap, re-orth, normalise)
// and one grid-wide "update" kernel (one warp per trailing column).
#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

constexpr int kPqSelThreads = 1024;
constexpr int kPqMaxK = 1024;

__global__ void pq_init_kernel(int64_t cols, int64_t rows, const double* __restrict__ Mt, int64_t ldmt,
                               double* __restrict__ WK, double* __restrict__ norms, int64_t* perm) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= cols) return;
  double a = 0.0;
  for (int64_t x = lane; x < rows; x += 32) {
    const double v = Mt[j * ldmt + x];
    WK[j * rows + x] = v;
    a = fma(v, v, a);
  }
  a = warp_sum(a);
  if (lane == 0) {
    norms[j] = sqrt(a);
    perm[j] = j;
  }
}

struct PqBest {
  double nrm;
  int64_t perm;
  int64_t j;
};

__device__ __forceinline__ bool pq_better(const PqBest& a, const PqBest& b) {
  return a.nrm > b.nrm || (a.nrm == b.nrm && a.perm < b.perm);
}

__device__ double pq_block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double acc = 0.0;
  for (int w = 0; w < nw; ++w) acc += red[w];
  return acc;
}

__global__ void __launch_bounds__(kPqSelThreads)
pq_select_kernel(int t, int k, int64_t cols, int64_t rows, double* __restrict__ WK, double* norms,
                 int64_t* perm, double* __restrict__ Qt, double* __restrict__ R, int64_t ldr,
                 int* status) {
  __shared__ double red[32];
  __shared__ PqBest bests[32];
  __shared__ double delta[kPqMaxK];
  __shared__ int64_t jstar_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  // ---- argmax over j in [t, cols) with the lowest-original-index tie-break
  PqBest b{-1.0, INT64_MAX, -1};
  for (int64_t j = t + tid; j < cols; j += blockDim.x) {
    PqBest c{norms[j], perm[j], j};
    if (pq_better(c, b)) b = c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    PqBest c{__shfl_xor_sync(0xffffffffu, b.nrm, o), __shfl_xor_sync(0xffffffffu, b.perm, o),
             __shfl_xor_sync(0xffffffffu, b.j, o)};
    if (pq_better(c, b)) b = c;
  }
  if (lane == 0) bests[warp] = b;
  __syncthreads();
  if (tid == 0) {
    PqBest bb = bests[0];
    for (int w = 1; w < nw; ++w)
      if (pq_better(bests[w], bb)) bb = bests[w];
    jstar_s = bb.j;
  }
  __syncthreads();
  const int64_t js = jstar_s;
  // ---- swap column t <-> js (work, R columns, perm, norms)
  if (js != t) {
    for (int64_t x = tid; x < rows; x += blockDim.x) {
      const double a = WK[(int64_t)t * rows + x];
      WK[(int64_t)t * rows + x] = WK[js * rows + x];
      WK[js * rows + x] = a;
    }
    for (int s = tid; s < k; s += blockDim.x) {
      const double a = R[(int64_t)s * ldr + t];
      R[(int64_t)s * ldr + t] = R[(int64_t)s * ldr + js];
      R[(int64_t)s * ldr + js] = a;
    }
    if (tid == 0) {
      const int64_t p = perm[t];
      perm[t] = perm[js];
      perm[js] = p;
      const double nn = norms[t];
      norms[t] = norms[js];
      norms[js] = nn;
    }
  }
  __syncthreads();
  double* v = Qt + (int64_t)t * rows;
  const double* wt = WK + (int64_t)t * rows;
  // ---- one classical re-orthogonalisation: delta = Q^T v; v -= Q delta
  if (t > 0) {
    for (int s = warp; s < t; s += nw) {
      double a = 0.0;
      for (int64_t x = lane; x < rows; x += 32) a = fma(Qt[(int64_t)s * rows + x], wt[x], a);
      a = warp_sum(a);
      if (lane == 0) delta[s] = a;
    }
    __syncthreads();
    for (int s = tid; s < t; s += blockDim.x) R[(int64_t)s * ldr + t] += delta[s];
    for (int64_t x = tid; x < rows; x += blockDim.x) {
      double acc = 0.0;
      for (int s = 0; s < t; ++s) acc = fma(Qt[(int64_t)s * rows + x], delta[s], acc);
      v[x] = wt[x] - acc;
    }
  } else {
    for (int64_t x = tid; x < rows; x += blockDim.x) v[x] = wt[x];
  }
  __syncthreads();
  double part = 0.0;
  for (int64_t x = tid; x < rows; x += blockDim.x) part = fma(v[x], v[x], part);
  const double pn = sqrt(pq_block_sum(part, red));
  if (pn != 0.0) {
    for (int64_t x = tid; x < rows; x += blockDim.x) v[x] = v[x] / pn;
  } else {
    // deterministic filler: first e_i whose residual against q_0..q_{t-1} has norm > 0.5
    bool found = false;
    for (int64_t i = 0; i < rows && !found; ++i) {
      double p2 = 0.0;
      for (int64_t x = tid; x < rows; x += blockDim.x) {
        double acc = (x == i) ? 1.0 : 0.0;
        for (int s = 0; s < t; ++s) acc -= Qt[(int64_t)s * rows + x] * Qt[(int64_t)s * rows + i];
        p2 = fma(acc, acc, p2);
      }
      const double nrm = sqrt(pq_block_sum(p2, red));
      if (nrm > 0.5) {
        for (int64_t x = tid; x < rows; x += blockDim.x) {
          double acc = (x == i) ? 1.0 : 0.0;
          for (int s = 0; s < t; ++s) acc -= Qt[(int64_t)s * rows + x] * Qt[(int64_t)s * rows + i];
          v[x] = acc / nrm;
        }
        found = true;
      }
    }
    if (!found && tid == 0) *status = SP_ENUMERICAL;
  }
  if (tid == 0) R[(int64_t)t * ldr + t] = pn;
}

// trailing columns j > t: coef = v . w_j ; R[t, j] = coef ; w_j -= coef v ; norm_j
__global__ void pq_update_kernel(int t, int64_t cols, int64_t rows, double* __restrict__ WK,
                                 double* __restrict__ norms, const double* __restrict__ Qt,
                                 double* __restrict__ R, int64_t ldr) {
  const int64_t j = t + 1 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= cols) return;
  const double* v = Qt + (int64_t)t * rows;
  double* w = WK + j * rows;
  double c = 0.0;
  for (int64_t x = lane; x < rows; x += 32) c = fma(v[x], w[x], c);
  c = warp_sum(c);
  double a = 0.0;
  for (int64_t x = lane; x < rows; x += 32) {
    const double nv = fma(-c, v[x], w[x]);
    w[x] = nv;
    a = fma(nv, nv, a);
  }
  a = warp_sum(a);
  if (lane == 0) {
    R[(int64_t)t * ldr + j] = c;
    norms[j] = sqrt(a);
  }
}

// Candidates of 1025 .. 4096 entries (cfg3: 5000 candidates of length 4096):
// one 128-thread CTA per candidate holds it in registers (PER values per
// thread), so the candidate is read once and written once -- the warp-per-
// candidate kernel above reads it a second time for the update, from L2 at
// best (164 MB of candidates against a 126 MB L2).  Same quantities, fixed
// summation order (thread-strided partials, warp shuffles, warps in order).
constexpr int kPqRegThreads = 128;

template <int PER>
__global__ void __launch_bounds__(kPqRegThreads)
pq_update_reg_kernel(int t, int64_t cols, int64_t rows, double* __restrict__ WK, double* __restrict__ norms,
                     const double* __restrict__ Qt, double* __restrict__ R, int64_t ldr) {
  __shared__ double red[2][kPqRegThreads / 32];
  const int64_t j = t + 1 + (int64_t)blockIdx.x;
  if (j >= cols) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* v = Qt + (int64_t)t * rows;
  double* w = WK + j * rows;
  double x[PER], vv[PER];
  double c = 0.0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int64_t e = tid + (int64_t)i * kPqRegThreads;
    x[i] = e < rows ? w[e] : 0.0;
    vv[i] = e < rows ? v[e] : 0.0;
    c = fma(vv[i], x[i], c);
  }
  c = warp_sum(c);
  if (lane == 0) red[0][warp] = c;
  __syncthreads();
  c = (red[0][0] + red[0][1]) + (red[0][2] + red[0][3]);
  double a = 0.0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int64_t e = tid + (int64_t)i * kPqRegThreads;
    const double nv = fma(-c, vv[i], x[i]);
    if (e < rows) w[e] = nv;
    a = fma(nv, nv, a);
  }
  a = warp_sum(a);
  if (lane == 0) red[1][warp] = a;
  __syncthreads();
  if (tid == 0) {
    R[(int64_t)t * ldr + j] = c;
    norms[j] = sqrt((red[1][0] + red[1][1]) + (red[1][2] + red[1][3]));
  }
}

// ------------------------------------------------------ long candidates ----
// Candidates much longer than their count (the ID of cfg5: 2000 candidates of
// length 262144): every step's work is spread over row blocks x column
// chunks with fixed-order partial reductions, instead of one warp (update)
// or one CTA (select / re-orthogonalisation) per candidate.  Same pivot rule
// and arithmetic (norms recomputed from the updated columns every step).
constexpr int kPlRows = 8192;   // rows per block (coefficient / update passes)
constexpr int kPlRowsV = 2048;  // rows per block (re-orthogonalisation passes: t dots per row)
constexpr int kPlCols = 16;     // candidates per update CTA
constexpr int kPlThreads = 256;

__device__ __forceinline__ double pl_block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double acc = 0.0;
#pragma unroll
  for (int w = 0; w < kPlThreads / 32; ++w) acc += red[w];
  return acc;
}

// argmax with the lowest-original-index tie-break, swap of the small state
// (perm, norms, R columns); the pivot index goes to *jsel
__global__ void __launch_bounds__(kPqSelThreads)
pl_select_kernel(int t, int k, int64_t cols, double* norms, int64_t* perm, double* R, int64_t ldr, int64_t* jsel) {
  __shared__ PqBest bests[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  PqBest b{-1.0, INT64_MAX, -1};
  for (int64_t j = t + tid; j < cols; j += blockDim.x) {
    PqBest c{norms[j], perm[j], j};
    if (pq_better(c, b)) b = c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    PqBest c{__shfl_xor_sync(0xffffffffu, b.nrm, o), __shfl_xor_sync(0xffffffffu, b.perm, o),
             __shfl_xor_sync(0xffffffffu, b.j, o)};
    if (pq_better(c, b)) b = c;
  }
  if (lane == 0) bests[warp] = b;
  __syncthreads();
  __shared__ int64_t js_s;
  if (tid == 0) {
    PqBest bb = bests[0];
    for (int w = 1; w < nw; ++w)
      if (pq_better(bests[w], bb)) bb = bests[w];
    js_s = bb.j;
    *jsel = bb.j;
  }
  __syncthreads();
  const int64_t js = js_s;
  if (js == t) return;
  for (int s2 = tid; s2 < k; s2 += blockDim.x) {
    const double a = R[(int64_t)s2 * ldr + t];
    R[(int64_t)s2 * ldr + t] = R[(int64_t)s2 * ldr + js];
    R[(int64_t)s2 * ldr + js] = a;
  }
  if (tid == 0) {
    const int64_t p = perm[t];
    perm[t] = perm[js];
    perm[js] = p;
    const double nn = norms[t];
    norms[t] = norms[js];
    norms[js] = nn;
  }
}

// row block rb: swap candidates t <-> *jsel, then partial[rb][s] = q_s . w_t (s < t)
__global__ void __launch_bounds__(kPlThreads)
pl_swap_dots_kernel(int t, int64_t rows, double* __restrict__ WK, const double* __restrict__ Qt,
                    const int64_t* __restrict__ jsel, double* __restrict__ partial,
                    const double* __restrict__ pend = nullptr) {
  __shared__ double red[kPlThreads / 32];
  const int64_t r0 = (int64_t)blockIdx.x * kPlRowsV, r1 = imin64(rows, r0 + kPlRowsV);
  const int64_t js = *jsel;
  double* wt = WK + (int64_t)t * rows;
  if (js != t) {
    double* wj = WK + js * rows;
    for (int64_t x = r0 + threadIdx.x; x < r1; x += kPlThreads) {
      const double a = wt[x];
      wt[x] = wj[x];
      wj[x] = a;
    }
    __syncthreads();
  }
  // lagged mode: update t - 1 is still pending on every trailing candidate; the
  // selected one (now at position t, its coefficient at R[t-1][t] after the
  // column swap) receives it here, the others in the fused pass of this step
  if (pend) {
    const double c = *pend;
    const double* vp = Qt + (int64_t)(t - 1) * rows;
    for (int64_t x = r0 + threadIdx.x; x < r1; x += kPlThreads) wt[x] = fma(-c, vp[x], wt[x]);
    __syncthreads();
  }
  // warp w takes s = w, w + 8, ...: no block barrier per dot product
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int s2 = warp; s2 < t; s2 += kPlThreads / 32) {
    const double* q = Qt + (int64_t)s2 * rows;
    double a0 = 0.0, a1 = 0.0;
    int64_t x = r0 + lane;
    for (; x + 32 < r1; x += 64) {
      a0 = fma(q[x], wt[x], a0);
      a1 = fma(q[x + 32], wt[x + 32], a1);
    }
    if (x < r1) a0 = fma(q[x], wt[x], a0);
    const double a = warp_sum(a0 + a1);
    if (lane == 0) partial[(int64_t)blockIdx.x * kPqMaxK + s2] = a;
  }
  (void)red;
}

// delta[s] = sum_rb partial[rb][s]; R[s][t] += delta[s]  (one CTA, fixed order)
__global__ void pl_delta_kernel(int t, int nb, const double* __restrict__ partial, double* __restrict__ delta,
                                double* __restrict__ R, int64_t ldr) {
  for (int s2 = threadIdx.x; s2 < t; s2 += blockDim.x) {
    double a = 0.0;
    for (int b = 0; b < nb; ++b) a += partial[(int64_t)b * kPqMaxK + s2];
    delta[s2] = a;
    R[(int64_t)s2 * ldr + t] += a;
  }
}

// v = w_t - sum_s delta_s q_s into Qt row t; part2[rb] = |v_rb|^2
__global__ void __launch_bounds__(kPlThreads)
pl_form_v_kernel(int t, int64_t rows, const double* __restrict__ WK, double* __restrict__ Qt,
                 const double* __restrict__ delta, double* __restrict__ part2) {
  __shared__ double red[kPlThreads / 32];
  __shared__ double ds[kPqMaxK];
  for (int s2 = threadIdx.x; s2 < t; s2 += kPlThreads) ds[s2] = delta[s2];
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * kPlRowsV, r1 = imin64(rows, r0 + kPlRowsV);
  const double* wt = WK + (int64_t)t * rows;
  double* v = Qt + (int64_t)t * rows;
  double p = 0.0;
  for (int64_t x = r0 + threadIdx.x; x < r1; x += kPlThreads) {
    double acc = 0.0;
    for (int s2 = 0; s2 < t; ++s2) acc = fma(Qt[(int64_t)s2 * rows + x], ds[s2], acc);
    const double vv = wt[x] - acc;
    v[x] = vv;
    p = fma(vv, vv, p);
  }
  p = pl_block_sum(p, red);
  if (threadIdx.x == 0) part2[blockIdx.x] = p;
}

// pn = sqrt(sum part2) (fixed order) -> R[t][t], pnv[0]; status 2 on a zero
// pivot (the caller redoes the factorisation on the per-candidate path,
// which owns the deterministic filler)
__global__ void pl_pivot_norm_kernel(int t, int nb, const double* __restrict__ part2, double* __restrict__ pnv,
                                     double* __restrict__ R, int64_t ldr, int* status) {
  if (threadIdx.x != 0) return;
  double a = 0.0;
  for (int b = 0; b < nb; ++b) a += part2[b];
  const double pn = sqrt(a);
  pnv[0] = pn;
  R[(int64_t)t * ldr + t] = pn;
  if (pn == 0.0) *status = 2;
}

__global__ void pl_normalise_kernel(int t, int64_t rows, double* __restrict__ Qt, const double* __restrict__ pnv) {
  const double pn = pnv[0];
  if (pn == 0.0) return;
  double* v = Qt + (int64_t)t * rows;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < rows; x += (int64_t)gridDim.x * blockDim.x)
    v[x] = v[x] / pn;
}

// pc[rb][j] = v_rb . w_j,rb for the CTA's candidate chunk (j > t)
__global__ void __launch_bounds__(kPlThreads)
pl_coef_kernel(int t, int64_t cols, int64_t rows, const double* __restrict__ WK, const double* __restrict__ Qt,
               double* __restrict__ pc) {
  __shared__ double red[kPlThreads / 32];
  const int64_t r0 = (int64_t)blockIdx.x * kPlRows, r1 = imin64(rows, r0 + kPlRows);
  const double* v = Qt + (int64_t)t * rows;
  const int64_t j0 = t + 1 + (int64_t)blockIdx.y * kPlCols;
  for (int u = 0; u < kPlCols; ++u) {
    const int64_t j = j0 + u;
    if (j >= cols) break;  // uniform
    const double* w = WK + j * rows;
    double a = 0.0;
    for (int64_t x = r0 + threadIdx.x; x < r1; x += kPlThreads) a = fma(v[x], w[x], a);
    a = pl_block_sum(a, red);
    if (threadIdx.x == 0) pc[(int64_t)blockIdx.x * cols + j] = a;
  }
}

// coef_j = sum_rb pc[rb][j] -> R[t][j], coef[j]
__global__ void pl_coef_reduce_kernel(int t, int nb, int64_t cols, const double* __restrict__ pc,
                                      double* __restrict__ coef, double* __restrict__ R, int64_t ldr) {
  const int64_t j = t + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  double a = 0.0;
  for (int b = 0; b < nb; ++b) a += pc[(int64_t)b * cols + j];
  coef[j] = a;
  R[(int64_t)t * ldr + j] = a;
}

// w_j -= coef_j v on the CTA's rows; pn2[rb][j] = |w_j,rb|^2 (updated)
__global__ void __launch_bounds__(kPlThreads)
pl_update_kernel(int t, int64_t cols, int64_t rows, double* __restrict__ WK, const double* __restrict__ Qt,
                 const double* __restrict__ coef, double* __restrict__ pn2) {
  __shared__ double red[kPlThreads / 32];
  const int64_t r0 = (int64_t)blockIdx.x * kPlRows, r1 = imin64(rows, r0 + kPlRows);
  const double* v = Qt + (int64_t)t * rows;
  const int64_t j0 = t + 1 + (int64_t)blockIdx.y * kPlCols;
  for (int u = 0; u < kPlCols; ++u) {
    const int64_t j = j0 + u;
    if (j >= cols) break;  // uniform
    double* w = WK + j * rows;
    const double c = coef[j];
    double a = 0.0;
    for (int64_t x = r0 + threadIdx.x; x < r1; x += kPlThreads) {
      const double nv = fma(-c, v[x], w[x]);
      w[x] = nv;
      a = fma(nv, nv, a);
    }
    a = pl_block_sum(a, red);
    if (threadIdx.x == 0) pn2[(int64_t)blockIdx.x * cols + j] = a;
  }
}

__global__ void pl_norms_kernel(int t, int nb, int64_t cols, const double* __restrict__ pn2, double* __restrict__ norms) {
  const int64_t j = t + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  double a = 0.0;
  for (int b = 0; b < nb; ++b) a += pn2[(int64_t)b * cols + j];
  norms[j] = sqrt(a);
}

// ---- lagged update: one read + write of the candidates per step instead of a read
// (coefficients) plus a read + write (update).
// Pass t applies the PENDING update t - 1 (coefficients in R[t-1][.]) in registers,
// writes the candidate back, and in the same pass takes its exact squared norm
// (pn2) and its dot with the new pivot direction v_t (pc).
__global__ void __launch_bounds__(kPlThreads)
pl_fused_kernel(int t, int64_t cols, int64_t rows, double* __restrict__ WK, const double* __restrict__ Qt,
                const double* __restrict__ Rprev, double* __restrict__ pc, double* __restrict__ pn2) {
  __shared__ double red[kPlThreads / 32];
  const int64_t r0 = (int64_t)blockIdx.x * kPlRows, r1 = imin64(rows, r0 + kPlRows);
  const double* v = Qt + (int64_t)t * rows;
  const double* vp = Rprev ? Qt + (int64_t)(t - 1) * rows : nullptr;
  const int64_t j0 = t + 1 + (int64_t)blockIdx.y * kPlCols;
  for (int u = 0; u < kPlCols; ++u) {
    const int64_t j = j0 + u;
    if (j >= cols) break;  // uniform
    double* w = WK + j * rows;
    double a = 0.0, n2 = 0.0;
    if (vp) {
      const double c = Rprev[j];
      for (int64_t x = r0 + threadIdx.x; x < r1; x += kPlThreads) {
        const double nv = fma(-c, vp[x], w[x]);
        w[x] = nv;
        n2 = fma(nv, nv, n2);
        a = fma(v[x], nv, a);
      }
    } else {
      for (int64_t x = r0 + threadIdx.x; x < r1; x += kPlThreads) {
        const double nv = w[x];
        n2 = fma(nv, nv, n2);
        a = fma(v[x], nv, a);
      }
    }
    a = pl_block_sum(a, red);
    n2 = pl_block_sum(n2, red);
    if (threadIdx.x == 0) {
      pc[(int64_t)blockIdx.x * cols + j] = a;
      pn2[(int64_t)blockIdx.x * cols + j] = n2;
    }
  }
}

// norms_j = sqrt(max(0, sum_rb pn2[rb][j] - coef_j^2)) for j > t: the residual
// norm after update t from the exact squared norm before it (the identity
// |w - c v|^2 = |w|^2 - c^2 holds for a unit v and c = v . w; rounding
// ~eps |w|^2 on the square)
__global__ void pl_downdate_kernel(int t, int nb, int64_t cols, const double* __restrict__ pn2,
                                   const double* __restrict__ coef, double* __restrict__ norms) {
  const int64_t j = t + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  double a = 0.0;
  for (int b = 0; b < nb; ++b) a += pn2[(int64_t)b * cols + j];
  const double e = fma(-coef[j], coef[j], a);
  norms[j] = e > 0.0 ? sqrt(e) : 0.0;
}

// the long-candidate factorisation loop; *fallback = true on a zero pivot
static int pivoted_qr_long(int64_t rows, int64_t cols, int k, double* WK, double* norms, int64_t* perm, double* Qt,
                           double* R, int64_t ldr, bool* fallback, cudaStream_t s) {
  *fallback = false;
  const int nb = ceil_div(rows, kPlRows), nbv = ceil_div(rows, kPlRowsV);
  Arena ar(s);
  SPB_ALLOC(ar, double, partial, (size_t)nbv * kPqMaxK);
  SPB_ALLOC(ar, double, part2, (size_t)nbv);
  SPB_ALLOC(ar, double, pc, (size_t)nb * cols);
  SPB_ALLOC(ar, double, coef, (size_t)cols);
  SPB_ALLOC(ar, double, delta, (size_t)kPqMaxK);
  SPB_ALLOC(ar, double, pnv, 1);
  SPB_ALLOC(ar, int64_t, jsel, 1);
  SPB_ALLOC(ar, int, status, 1);
  SPB_CUDA(cudaMemsetAsync(status, 0, sizeof(int), s));
  // lagged update (default; SPB_PQ_EAGER=1: the three-pass step, for comparison):
  // cfg5 power_id 485 -> 447 ms, same pivots / P / reconstruction error
  static const bool lagged = getenv("SPB_PQ_EAGER") == nullptr;
  double* pn2l = nullptr;
  if (lagged) {
    pn2l = ar.alloc<double>((size_t)nb * cols);
    if (!pn2l) {
      set_error("pivoted QR workspace allocation failed");
      return SP_ECUDA;
    }
  }
  for (int t = 0; t < k; ++t) {
    pl_select_kernel<<<1, kPqSelThreads, 0, s>>>(t, k, cols, norms, perm, R, ldr, jsel);
    pl_swap_dots_kernel<<<nbv, kPlThreads, 0, s>>>(t, rows, WK, Qt, jsel, partial,
                                                   lagged && t > 0 ? R + (int64_t)(t - 1) * ldr + t : nullptr);
    if (t > 0) pl_delta_kernel<<<1, 128, 0, s>>>(t, nbv, partial, delta, R, ldr);
    pl_form_v_kernel<<<nbv, kPlThreads, 0, s>>>(t, rows, WK, Qt, delta, part2);
    pl_pivot_norm_kernel<<<1, 32, 0, s>>>(t, nbv, part2, pnv, R, ldr, status);
    pl_normalise_kernel<<<std::min<int64_t>(4 * kNumSMs, ceil_div(rows, 256)), 256, 0, s>>>(t, rows, Qt, pnv);
    count_launch(t > 0 ? 6 : 5);
    const int64_t trail = cols - t - 1;
    if (trail > 0) {
      dim3 g(nb, ceil_div(trail, kPlCols));
      if (lagged) {
        pl_fused_kernel<<<g, kPlThreads, 0, s>>>(t, cols, rows, WK, Qt, t > 0 ? R + (int64_t)(t - 1) * ldr : nullptr,
                                                 pc, pn2l);
        pl_coef_reduce_kernel<<<ceil_div(trail, 256), 256, 0, s>>>(t, nb, cols, pc, coef, R, ldr);
        pl_downdate_kernel<<<ceil_div(trail, 256), 256, 0, s>>>(t, nb, cols, pn2l, coef, norms);
        count_launch(3);
        SPB_CHECK_LAUNCH();
        continue;
      }
      pl_coef_kernel<<<g, kPlThreads, 0, s>>>(t, cols, rows, WK, Qt, pc);
      pl_coef_reduce_kernel<<<ceil_div(trail, 256), 256, 0, s>>>(t, nb, cols, pc, coef, R, ldr);
      pl_update_kernel<<<g, kPlThreads, 0, s>>>(t, cols, rows, WK, Qt, coef, pc);
      pl_norms_kernel<<<ceil_div(trail, 256), 256, 0, s>>>(t, nb, cols, pc, norms);
      count_launch(4);
    }
    SPB_CHECK_LAUNCH();
  }
  int hst = 0;
  SPB_TRY(read_small(&hst, status, sizeof(int), s));
  *fallback = hst != 0;
  return SP_OK;
}

int pivoted_qr(int64_t rows, int64_t cols, const double* Mt, int64_t ldmt, int k, int64_t* perm,
               double* Q, int64_t ldq, double* R, int64_t ldr, cudaStream_t s) {
  SPB_REQUIRE(k >= 1 && k <= std::min(rows, cols),
              "rank k=" + std::to_string(k) + " outside [1, " + std::to_string(std::min(rows, cols)) + "]");
  SPB_REQUIRE(k <= kPqMaxK, "pivoted_qr supports k <= 1024");
  SPB_REQUIRE(ldmt >= rows && ldr >= cols && ldq >= k, "bad pivoted_qr leading dimension");
  SPB_TRY(check_finite(cols, rows, Mt, ldmt, "pivoted QR input contains non-finite entries", s));
  Arena ar(s);
  SPB_ALLOC(ar, double, WK, (size_t)cols * rows);
  SPB_ALLOC(ar, double, norms, (size_t)cols);
  SPB_ALLOC(ar, double, Qt, (size_t)k * rows);
  SPB_ALLOC(ar, int, status, 1);
  SPB_CUDA(cudaMemsetAsync(status, 0, sizeof(int), s));
  SPB_CUDA(cudaMemset2DAsync(R, ldr * sizeof(double), 0, cols * sizeof(double), k, s));
  pq_init_kernel<<<ceil_div(cols * 32, 256), 256, 0, s>>>(cols, rows, Mt, ldmt, WK, norms, perm);
  count_launch();
  SPB_CHECK_LAUNCH();
  bool done = false;
  if (rows >= 4 * kPlRows && rows >= 8 * cols) {
    bool fb = false;
    SPB_TRY(pivoted_qr_long(rows, cols, k, WK, norms, perm, Qt, R, ldr, &fb, s));
    done = !fb;
    if (fb) {  // zero pivot: restart on the per-candidate path (deterministic filler)
      SPB_CUDA(cudaMemset2DAsync(R, ldr * sizeof(double), 0, cols * sizeof(double), k, s));
      pq_init_kernel<<<ceil_div(cols * 32, 256), 256, 0, s>>>(cols, rows, Mt, ldmt, WK, norms, perm);
      count_launch();
      SPB_CHECK_LAUNCH();
    }
  }
  for (int t = 0; t < k && !done; ++t) {
    pq_select_kernel<<<1, kPqSelThreads, 0, s>>>(t, k, cols, rows, WK, norms, perm, Qt, R, ldr, status);
    count_launch();
    SPB_CHECK_LAUNCH();
    if (t + 1 < cols) {
      const unsigned nc = (unsigned)(cols - t - 1);
      if (rows > 2048 && rows <= 4096)
        pq_update_reg_kernel<32><<<nc, kPqRegThreads, 0, s>>>(t, cols, rows, WK, norms, Qt, R, ldr);
      else if (rows > 1024 && rows <= 2048)
        pq_update_reg_kernel<16><<<nc, kPqRegThreads, 0, s>>>(t, cols, rows, WK, norms, Qt, R, ldr);
      else
        pq_update_kernel<<<ceil_div((cols - t - 1) * 32, 256), 256, 0, s>>>(t, cols, rows, WK, norms, Qt, R, ldr);
      count_launch();
      SPB_CHECK_LAUNCH();
    }
  }
  int hst = 0;
  SPB_TRY(read_small(&hst, status, sizeof(int), s));
  if (hst != 0) {
    set_error("cannot extend orthonormal basis");
    return SP_ENUMERICAL;
  }
  SPB_TRY(transpose(k, rows, Qt, rows, Q, ldq, s));
  SPB_TRY(sign_fix(rows, k, Q, ldq, R, ldr, cols, true, s));
  return SP_OK;
}

}  // namespace spb
