// Householder-reconstruction completion (complete.cu header comment), as a
// device function shared by complete.cu and finish.cu.
#pragma once
#include "common.cuh"

namespace spb {

// workspace
constexpr int kHcMaxR = 32;
constexpr int kHcMaxK = 256;
struct HcShared {
  double W[kHcMaxR][kHcMaxR + 1];   // LU workspace -> L1 (strict lower) + U (upper)
  double Ui[kHcMaxR][kHcMaxR + 1];  // U^{-1}
  double Li[kHcMaxR][kHcMaxR + 1];  // L1^{-1}
  double T[kHcMaxR][kHcMaxR + 1];
  double G[kHcMaxR][kHcMaxR + 1];   // U^{-1} T U^{-T}
  double S[kHcMaxR];
};
// in: Qtop = Q[0:k, 0:r] (ld ldq).  out: Kp (r x (k-r), ld kr) and the top k
// rows of the completion block E' (k x (k-r), ld lde).  Executed by threads
// [0, nt) of a group (tid = rank in the group); every group of the CTA must
// run it with the same r and k (the __syncthreads are CTA-wide), so two
// groups can complete two bases at once (finish.cu).
static __device__ __noinline__ void hh_complete_dev(int r, int k, const double* __restrict__ Q, int64_t ldq, double* __restrict__ Kp,
                                double* __restrict__ Etop, int64_t lde, const double* __restrict__ B, int64_t ldb,
                                double* __restrict__ Mf, double* __restrict__ Etf, HcShared& sh, int tid, int nt) {
  double(*W)[kHcMaxR + 1] = sh.W;
  double(*Ui)[kHcMaxR + 1] = sh.Ui;
  double(*Li)[kHcMaxR + 1] = sh.Li;
  double(*T)[kHcMaxR + 1] = sh.T;
  double(*G)[kHcMaxR + 1] = sh.G;
  double* S = sh.S;
  const int kr = k - r;
  for (int e = tid; e < r * r; e += nt) W[e / r][e % r] = Q[(int64_t)(e / r) * ldq + (e % r)];
  __syncthreads();
  // LU without pivoting of Q1 - S, S_i = -sign(current pivot)
  for (int i = 0; i < r; ++i) {
    if (tid == 0) {
      const double s = W[i][i] >= 0.0 ? -1.0 : 1.0;
      S[i] = s;
      W[i][i] -= s;
    }
    __syncthreads();
    const double piv = W[i][i];
    for (int e = tid; e < (r - i - 1) * (r - i); e += nt) {
      const int a = i + 1 + e / (r - i), b = i + e % (r - i);
      if (b == i) continue;
      W[a][b] = fma(-W[a][i] / piv, W[i][b], W[a][b]);
    }
    __syncthreads();
    for (int a = i + 1 + tid; a < r; a += nt) W[a][i] /= piv;  // L multipliers
    __syncthreads();
  }
  // U^{-1} (upper) and L1^{-1} (unit lower), one column per thread
  for (int col = tid; col < r; col += nt) {
    for (int a = r - 1; a >= 0; --a) {
      double acc = (a == col) ? 1.0 : 0.0;
      for (int b = a + 1; b < r; ++b) acc = fma(-W[a][b], Ui[b][col], acc);
      Ui[a][col] = (a <= col) ? acc / W[a][a] : 0.0;
    }
    for (int a = 0; a < r; ++a) {
      double acc = (a == col) ? 1.0 : 0.0;
      for (int b = 0; b < a; ++b) acc = fma(-W[a][b], Li[b][col], acc);
      Li[a][col] = (a >= col) ? acc : 0.0;
    }
  }
  __syncthreads();
  // T = -U S L1^{-T}
  for (int e = tid; e < r * r; e += nt) {
    const int a = e / r, b = e % r;
    double acc = 0.0;
    for (int q = a; q < r; ++q) acc = fma(W[a][q] * S[q], Li[b][q], acc);  // U[a][q] S_q (L1^{-T})[q][b]
    T[a][b] = -acc;
  }
  __syncthreads();
  // K' = U^{-1} T L2top^T with L2top = Q[r:k] U^{-1}  =>  K' = G Q[r:k]^T,
  // G = U^{-1} T U^{-T}.  First Li <- T U^{-T} (Li is free now), then G.
  for (int e = tid; e < r * r; e += nt) {
    const int a = e / r, b = e % r;
    double acc = 0.0;
    for (int q = b; q < r; ++q) acc = fma(T[a][q], Ui[b][q], acc);  // (U^{-T})[q][b] = Ui[b][q]
    Li[a][b] = acc;
  }
  __syncthreads();
  for (int e = tid; e < r * r; e += nt) {
    const int a = e / r, b = e % r;
    double acc = 0.0;
    for (int q = a; q < r; ++q) acc = fma(Ui[a][q], Li[q][b], acc);
    G[a][b] = acc;
  }
  __syncthreads();
  for (int e = tid; e < r * kr; e += nt) {
    const int a = e / kr, j = e % kr;
    double acc = 0.0;
    for (int p = 0; p < r; ++p) acc = fma(G[a][p], Q[(int64_t)(r + j) * ldq + p], acc);
    Kp[(int64_t)a * kr + j] = acc;
    Etop[(int64_t)a * lde + j] = S[a] * acc;  // rows 0..r-1 of E'
  }
  for (int e = tid; e < kr * kr; e += nt) {
    const int a = e / kr, j = e % kr;
    Etop[(int64_t)(r + a) * lde + j] = (a == j) ? 1.0 : 0.0;  // rows r..k-1 of E'
  }
  if (B == nullptr) return;
  // fused product (product_with_completion): Mf = [B | -B Kp], Etf = [0 | E']
  __syncthreads();  // Kp / Etop (global) written by this CTA above
  for (int e = tid; e < r * k; e += nt) {
    const int i = e / k, j = e % k;
    double v;
    if (j < r) {
      v = B[(int64_t)i * ldb + j];
    } else {
      double a = 0.0;
      for (int q = 0; q < r; ++q) a = fma(B[(int64_t)i * ldb + q], Kp[q * kr + (j - r)], a);
      v = -a;
    }
    Mf[e] = v;
  }
  for (int e = tid; e < k * k; e += nt) {
    const int i = e / k, j = e % k;
    Etf[e] = j < r ? 0.0 : Etop[(int64_t)i * lde + (j - r)];
  }
}


}  // namespace spb
