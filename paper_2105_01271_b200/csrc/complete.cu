// Orthonormal completion of an orthonormal block without a QR: Householder
// reconstruction (Ballard, Demmel, Grigori, Jacquelin, Nguyen, Solomonik,
// "Reconstructing Householder vectors from tall-skinny QR", 2014).
//
// For Q (N x r) with orthonormal columns, the LU factorisation without
// pivoting  Q - [S; 0] = Y U  (S = diag(+-1) chosen so every pivot has
// magnitude >= 1) gives the compact-WY orthogonal H = I - Y T Y^T with
// T = -U S Y1^{-T} and H [S; 0] = Q.  Columns r..k-1 of H are therefore an
// orthonormal completion of span(Q):
//     H e_j = e_j - Y T Y_j^T  =  E' - Q K'
// with K' = U^{-1} T L2top^T (r x (k-r)), L2top = Q[r:k] U^{-1}, and E' zero
// except rows 0..r-1 (= S K') and rows r..k-1 (= I).  Everything but the
// final N x r x (k-r) GEMM lives in the top k rows of Q: one small kernel.
// Replaces the QR of [Q | random] the padding of U, V to rank k needed
// (the reference's rank-k shape contract, tests/test_svd.py:163-171).
#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"
#include "hh_complete.cuh"

namespace spb {


__global__ void __launch_bounds__(256)
hh_complete_kernel(int r, int k, const double* __restrict__ Q, int64_t ldq, double* __restrict__ Kp,
                   double* __restrict__ Etop, int64_t lde, const double* __restrict__ B = nullptr,
                   int64_t ldb = 0, double* __restrict__ Mf = nullptr, double* __restrict__ Etf = nullptr) {
  __shared__ HcShared sh;
  hh_complete_dev(r, k, Q, ldq, Kp, Etop, lde, B, ldb, Mf, Etf, sh, threadIdx.x, blockDim.x);
}

// out (N x k, ld ldo): columns [0, r) orthonormal on entry; columns [r, k)
// receive the Householder completion.  Returns SP_ECONFIG (caller falls back)
// when r or k exceed the small-kernel limits.
int householder_complete(int64_t N, int r, int k, double* out, int64_t ldo, cudaStream_t s,
                         double* kp_out) {
  if (r >= k) return SP_OK;
  if (r > kHcMaxR || k > kHcMaxK || N < k) {
    set_error("householder_complete limits exceeded");
    return SP_ECONFIG;
  }
  const int kr = k - r;
  if (r == 0) {
    // H = I: the first k columns of the identity
    SPB_CUDA(cudaMemset2DAsync(out, ldo * sizeof(double), 0, kr * sizeof(double), N, s));
    SPB_TRY(fill_identity(k, out, ldo, s));
    return SP_OK;
  }
  Arena ar(s);
  SPB_ALLOC(ar, double, Kp, (size_t)r * kr);
  if (r * kr <= 64 * 64 && kr <= 256) {
    // out[:, r:k] = E' - Q K' in one streaming pass (E' added on the top k rows)
    SPB_ALLOC(ar, double, Et, (size_t)k * kr);
    hh_complete_kernel<<<1, 256, 0, s>>>(r, k, out, ldo, kp_out ? kp_out : Kp, Et, kr);
    count_launch();
    SPB_CHECK_LAUNCH();
    return tall_mul(N, r, out, ldo, kr, kp_out ? kp_out : Kp, kr, -1.0, 0.0, out + r, ldo, s, Et, kr, k);
  }
  // zero the completion block, then write its top k rows (E') in place
  SPB_CUDA(cudaMemset2DAsync(out + r, ldo * sizeof(double), 0, kr * sizeof(double), N, s));
  hh_complete_kernel<<<1, 256, 0, s>>>(r, k, out, ldo, Kp, out + r, ldo);
  count_launch();
  SPB_CHECK_LAUNCH();
  // sharded callers: the other row blocks of the completion are -Q_i K'
  if (kp_out) SPB_CUDA(cudaMemcpyAsync(kp_out, Kp, (size_t)r * kr * sizeof(double), cudaMemcpyDeviceToDevice, s));
  // out[:, r:k] = E' - Q K'
  return gemm(0, 0, N, kr, r, -1.0, out, ldo, Kp, kr, 1.0, out + r, ldo, s);
}

// out (N x k) = [X B | completion]: the kept factor X B (X: N x r, B: r x r)
// and its Householder completion written in ONE streaming pass over the N
// rows (out = X [B | -B K'] + [0 | E'] on the top k rows).  K' only needs the
// top k rows of X B, formed first.  Returns SP_ECONFIG (caller falls back to
// product + householder_complete) outside the small-kernel limits.
bool product_with_completion_ok(int64_t N, int r, int k) {
  return !(r < 1 || r >= k || r > kHcMaxR || k > kHcMaxK || N < k || r * k > 64 * 64 || k > 256);
}

int product_with_completion(int64_t N, int r, int k, const double* X, int64_t ldx, const double* B, int64_t ldb,
                            double* out, int64_t ldo, cudaStream_t s) {
  const int kr = k - r;
  if (!product_with_completion_ok(N, r, k)) {
    set_error("product_with_completion limits exceeded");
    return SP_ECONFIG;
  }
  Arena ar(s);
  SPB_ALLOC(ar, double, Kp, (size_t)r * kr);
  SPB_ALLOC(ar, double, Et, (size_t)k * kr);
  SPB_ALLOC(ar, double, Mf, (size_t)r * k);
  SPB_ALLOC(ar, double, Etf, (size_t)k * k);
  SPB_TRY(gemm(0, 0, k, r, r, 1.0, X, ldx, B, ldb, 0.0, out, ldo, s));  // top k rows of X B
  hh_complete_kernel<<<1, 256, 0, s>>>(r, k, out, ldo, Kp, Et, kr, B, ldb, Mf, Etf);
  count_launch();
  SPB_CHECK_LAUNCH();
  return tall_mul(N, r, X, ldx, k, Mf, k, 1.0, 0.0, out, ldo, s, Etf, k, k);
}

__global__ void fill_identity_kernel(int k, double* out, int64_t ldo) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) out[(int64_t)i * ldo + i] = 1.0;
}

int fill_identity(int k, double* out, int64_t ldo, cudaStream_t s) {
  fill_identity_kernel<<<ceil_div(k, 128), 128, 0, s>>>(k, out, ldo);
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

}  // namespace spb
