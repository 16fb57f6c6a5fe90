// Internal (C++) entry points of the device library; the C-ABI in capi.cu
// wraps these.  All take a cudaStream_t and return an SP_* status.
#pragma once
#include <vector>

#include "common.cuh"

namespace spb {

int apply_stencil(const void* A, int a_dtype, int64_t rows, int64_t n, int64_t lda,
                  const int64_t* idx, const double* w, int depth, int64_t nc, bool exact,
                  double* out, int64_t ldo, cudaStream_t s);
int check_columns(const int64_t* cols, int64_t count, int64_t n, cudaStream_t s);
int skinny_atz(const void* A, int a_dtype, int64_t m, int64_t n, int64_t lda, const double* Z,
               int64_t ldz, int r, double* Y, int64_t ldy, cudaStream_t s);
int gemm(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
         int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
         cudaStream_t s);
int tsqr(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
         double* R, int64_t ldr, cudaStream_t s);
// TSQR of a <= 32-column block in two phases: the leaf tree (R), then Q
struct TsqrPlan {
  struct Level {
    int64_t rows = 0;
    int nch = 0, cl = 0;
    int ch = 256;  // rows per CTA of the level's leaf kernel
    double* V = nullptr;
    double* T = nullptr;
    double* Rs = nullptr;
  };
  std::vector<Level> lv;
  double* sgn = nullptr;
  double* Mg = nullptr;  // single-chunk root: M = T V_top^T diag(sgn)
  int cols = 0;
};
// gemm() computing only the tiles on and above the diagonal of a square C (the
// caller mirrors: mirror_upper), for products known to be symmetric
int gemm_upper(int ta, int tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
               const double* B, int64_t ldb, double beta, double* C, int64_t ldc, cudaStream_t s);
int mirror_upper(int64_t n, double* W, int64_t ldw, cudaStream_t s);
// W = A A^T (M x M) from the tiles on and above the diagonal, mirrored
int gemm_aat(int64_t M, int64_t K, const double* A, int64_t lda, double* W, int64_t ldw, cudaStream_t s);
int tsqr_factor(int64_t rows, int cols, const double* X, int64_t ldx, double* R, int64_t ldr, TsqrPlan& plan,
                Arena& ar, cudaStream_t s);
int tsqr_form_q(const TsqrPlan& plan, double* Q, int64_t ldq, Arena& ar, cudaStream_t s);
// R (b x b upper) with R^T R = X^T X from a double-double Gram (b <= 32)
bool gram_chol_dd_ok(int64_t rows, int b);
int gram_chol_dd(int64_t rows, int b, const double* X, int64_t ldx, double* R, int64_t ldr, Arena& ar,
                 cudaStream_t s, int nslab = 1, int64_t slab_stride = 0);
// op(A) (B_hi + B_lo) nearly exactly rounded (Ozaki slices on DMMA): C_hi (+ C_lo)
int gemm_exact(int ta, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B_hi,
               const double* B_lo, int64_t ldb, double* C_hi, double* C_lo, int64_t ldc, cudaStream_t s,
               bool symmetric = false);
void ozaki_plan(int64_t K, int* bits, int* nsl);
int row_exponents(int64_t rows, int64_t cols, const double* X, int64_t ldx, int* e, cudaStream_t s);
int col_exponents(int64_t rows, int64_t cols, const double* X, int64_t ldx, int* e, cudaStream_t s);
int gemm_exact_levels(int ta, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const int* ea,
                      const double* B, int64_t ldb, const int* eb, int bits, int nsl, double* Lv, cudaStream_t s,
                      bool symmetric = false);
int dd_levels(int64_t M, int64_t N, const double* Lv, int nsl, const double* tail, double* hi, double* lo,
              int64_t ldc, cudaStream_t s);
// sharded pivoted QR steps (pivqr_dist.cu) and the ID coefficients from a QR
int pqd_begin(int64_t m, int64_t len, int k, const double* E, int64_t lde, double* WK, int64_t* perm, double* R,
              int64_t ldr, double* pn2, cudaStream_t s);
int pqd_select(int t, int k, int64_t m, int64_t len, const double* n2, int64_t* perm, double* R, int64_t ldr,
               double* WK, const double* Qt, double* delta, int64_t* jsel, cudaStream_t s);
int pqd_orth(int t, int64_t len, const double* delta, double* R, int64_t ldr, const double* WK, double* Qt,
             double* part2, cudaStream_t s);
int pqd_coef(int t, int64_t m, int64_t len, const double* p2, double* R, int64_t ldr, const double* WK, double* Qt,
             double* coef, int* status, cudaStream_t s);
int pqd_update(int t, int64_t m, int64_t len, const double* coef, double* R, int64_t ldr, double* WK, const double* Qt,
               double* pn2, cudaStream_t s);
int id_from_qr(int64_t m, int k, const int64_t* perm, const double* R, int64_t ldr, double* P, int64_t* indices,
               int* warn, cudaStream_t s);
int gemm_partials(int ta, int tb, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                  int64_t ldb, Arena& ar, double** P, int* S_out, cudaStream_t s);
int tall_gram(int64_t rows, int c, const double* X, int64_t ldx, int d, const double* Y, int64_t ldy,
              double alpha, double beta, double* G, int64_t ldg, cudaStream_t s);
int tall_gram_partials(int64_t rows, int c, const double* X, int64_t ldx, int d, const double* Y, int64_t ldy,
                       double* part, int nb_max, int* nb_out, cudaStream_t s);
// C (M x N, ldc) = alpha * sum_{s < S} P[s] + beta * C, P dense M x N slabs, fixed order
int split_reduce(const double* P, int S, int64_t M, int64_t N, double alpha, double beta, double* C, int64_t ldc,
                 cudaStream_t s);
// O = alpha X M + beta O (+ top[row] for row < top_rows); O may alias X's rows
int tall_mul(int64_t rows, int c, const double* X, int64_t ldx, int d, const double* M, int64_t ldm, double alpha,
             double beta, double* O, int64_t ldo, cudaStream_t s, const double* top = nullptr, int64_t ldt = 0,
             int64_t top_rows = 0);
int cholqr2_async(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
                  double* R, int64_t ldr, int* dflag, cudaStream_t s);
int check_finite_async(int64_t rows, int64_t cols, const double* X, int64_t ldx, int* dflag, cudaStream_t s);
int cholqr2(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
            double* R, int64_t ldr, bool* breakdown, cudaStream_t s);
int qr_tall(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq, double* R,
            int64_t ldr, bool well_conditioned, cudaStream_t s);
int jacobi_svd(int64_t n, const double* M, int64_t ldm, double* U, int64_t ldu, double* S,
               double* V, int64_t ldv, cudaStream_t s);
int jacobi_svd_tr(int64_t n, const double* M, int64_t ldm, bool trans, double* U, int64_t ldu, double* S,
                  double* V, int64_t ldv, cudaStream_t s);
int transpose(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Y, int64_t ldy,
              cudaStream_t s);
int copy2d(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Y, int64_t ldy,
           cudaStream_t s);
int fill_uniform(int64_t rows, int64_t cols, double* X, int64_t ldx, uint64_t seed, cudaStream_t s,
                 int64_t row_offset = 0);
int householder_complete(int64_t N, int r, int k, double* out, int64_t ldo, cudaStream_t s,
                         double* kp_out = nullptr);
int fill_identity(int k, double* out, int64_t ldo, cudaStream_t s);
int complete_basis(int64_t N, int r, int k, double* out, int64_t ldo, uint64_t seed, cudaStream_t s);
bool product_with_completion_ok(int64_t N, int r, int k);
int product_with_completion(int64_t N, int r, int k, const double* X, int64_t ldx, const double* B, int64_t ldb,
                            double* out, int64_t ldo, cudaStream_t s);
int max_abs(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* out, cudaStream_t s);
int fill_uniform_scaled(int64_t rows, int64_t cols, double* X, int64_t ldx, uint64_t seed, const double* scale,
                        double factor, cudaStream_t s);
int scale_cols(int64_t rows, int64_t cols, double* X, int64_t ldx, const double* d, cudaStream_t s);
int check_finite(int64_t rows, int64_t cols, const double* X, int64_t ldx, const char* what,
                 cudaStream_t s);
int sign_fix(int64_t rows, int64_t cols, double* basis, int64_t ldb, double* comp, int64_t ldc,
             int64_t comp_len, bool comp_row, cudaStream_t s);
int pinv_apply(const double* s, int64_t n, double tol, double* out, cudaStream_t st);
int trsm_upper(int64_t k, const double* R, int64_t ldr, int64_t ncols, const double* B, int64_t ldb,
               double* X, int64_t ldx, cudaStream_t s);
int thin_qr(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
            double* R, int64_t ldr, cudaStream_t s);
int thin_svd(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* U, int64_t ldu,
             double* S, double* V, int64_t ldv, cudaStream_t s);
int thin_svd_t(int64_t rows, int64_t cols, const double* Xt, int64_t ldxt, double* U, int64_t ldu, double* S,
               double* V, int64_t ldv, cudaStream_t s);
int scale_columns(int64_t rows, int64_t cols, double* X, int64_t ldx, const double* d, bool divide, cudaStream_t s);
int gather_rows(const void* X, int dtype, int64_t ldx, int64_t cols, const int64_t* idx, int64_t k, double* out,
                int64_t ldo, cudaStream_t s);
int pivoted_qr(int64_t rows, int64_t cols, const double* Mt, int64_t ldmt, int k, int64_t* perm,
               double* Q, int64_t ldq, double* R, int64_t ldr, cudaStream_t s);
int frob_residual(const void* A, int a_dtype, int64_t m, int64_t n, int64_t lda, const double* U,
                  int64_t ldu, const double* S, const double* V, int64_t ldv, int k, double* out2,
                  cudaStream_t s);

}  // namespace spb
