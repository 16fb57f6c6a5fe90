// extern "C" boundary (include/sketchpress_b200.h).  Thin wrappers that cast
// the stream, keep the thread-local error string and the launch counter.
#include <string>

#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

static thread_local std::string g_err;
static thread_local int64_t g_launches = 0;

void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }
void count_launch(int n) { g_launches += n; }
int64_t launches() { return g_launches; }

int single_pass_svd(const void* A, int a_dtype, int64_t m, int64_t n, int64_t lda, const int64_t* idx,
                    const double* w, int depth, int64_t nc, const double* omega, int64_t ell, int k,
                    const double* pre_s0, double* U, double* S, double* V, int64_t* info,
                    cudaStream_t s);
int power_svd(const void* A, int a_dtype, int64_t m, int64_t n, int64_t lda, const int64_t* idx,
              const double* w, int depth, int64_t nc, const double* omega, int64_t ell,
              const int64_t* cols, int64_t ncols, int q, int k, const double* pre_s0,
              const double* pre_c, int hints, double* U, double* S, double* V, int64_t* info, cudaStream_t s);
int power_id(const void* A, int a_dtype, int64_t m, int64_t n, int64_t lda, const int64_t* idx,
             const double* w, int depth, int64_t nc, const int64_t* cols, int64_t ncols, int q, int k,
             int r_req, const double* proj, int64_t proj_ell, int id_on_basis, const double* pre_s0,
             const double* pre_c, double* P, int64_t* indices, double* skeleton, double* lift_left,
             double* lift_right, double* lift_ur, int r_max, int64_t* info, cudaStream_t s);
int row_id(int64_t m, int64_t cols, const double* M, int64_t ldm, int k, double* P, int64_t* indices,
           int* warn, cudaStream_t s);
int deferred_status(int* out);
int srht_sketch(int64_t rows, int64_t cols, const double* X, int64_t ldx, int b, uint64_t seed, double* Y,
                int64_t ldy, int* flag, cudaStream_t s);
int srht_gather(const void* A, int a_dtype, int64_t rows, int64_t lda, const int64_t* gidx, int64_t cols, double* C,
                int64_t ldc, int b, uint64_t seed, double* Y, int64_t ldy, int* flag, cudaStream_t s);
std::string host_trace_dump();
void set_finish_mode(int mode);
int sketch_basis(const double* X, int64_t rows, int64_t cols, int64_t ldx, double power, int r_max, double* U,
                 int64_t ldu, double* S, int64_t* info, cudaStream_t s);

}  // namespace spb

using namespace spb;

#define ST(x) reinterpret_cast<cudaStream_t>(x)

extern "C" {

int sp_abi_version(void) { return SP_ABI_VERSION; }
const char* sp_last_error(void) { return last_error(); }
int64_t sp_launch_count(void) { return launches(); }
int sp_release_workspaces(void) {
  ws_release_all();
  int d = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&d) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess)
    cudaMemPoolTrimTo(pool, 0);
  cudaGetLastError();
  return SP_OK;
}
int sp_deferred_status(int32_t* flag) {
  int f = 0;
  const int st = deferred_status(&f);
  *flag = f;
  return st;
}
// diagnostics: the host-side trace (SPB_HOST_TRACE=1) as text; not in the header
const char* sp_host_trace(void) {
  static thread_local std::string t;
  t = host_trace_dump();
  return t.c_str();
}
int sp_set_finish_mode(int32_t mode) {
  set_finish_mode(mode);
  return SP_OK;
}

int sp_apply_stencil(const void* A, int32_t a_dtype, int64_t rows, int64_t n, int64_t lda,
                     const int64_t* idx, const double* w, int32_t depth, int64_t n_c,
                     int32_t exact_copy, double* out, int64_t ldo, void* stream) {
  return apply_stencil(A, a_dtype, rows, n, lda, idx, w, depth, n_c, exact_copy != 0, out, ldo, ST(stream));
}

int sp_check_columns(const int64_t* cols, int64_t count, int64_t n, void* stream) {
  return check_columns(cols, count, n, ST(stream));
}

int sp_skinny_atz(const void* A, int32_t a_dtype, int64_t m, int64_t n, int64_t lda, const double* Z,
                  int64_t ldz, int32_t r, double* Y, int64_t ldy, void* stream) {
  return skinny_atz(A, a_dtype, m, n, lda, Z, ldz, r, Y, ldy, ST(stream));
}

int sp_gemm(int32_t trans_a, int32_t trans_b, int64_t M, int64_t N, int64_t K, double alpha,
            const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
            int64_t ldc, void* stream) {
  return gemm(trans_a, trans_b, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ST(stream));
}

int sp_gemm_aat(int64_t M, int64_t K, const double* A, int64_t lda, double* W, int64_t ldw, void* stream) {
  return gemm_aat(M, K, A, lda, W, ldw, ST(stream));
}

int sp_gemm_exact(int32_t trans_a, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                  const double* B_hi, const double* B_lo, int64_t ldb, double* C_hi, double* C_lo,
                  int64_t ldc, void* stream) {
  return gemm_exact(trans_a, M, N, K, A, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, ST(stream));
}

int sp_exact_plan(int64_t K, int32_t* bits, int32_t* nsl) {
  if (K < 1 || !bits || !nsl) {
    set_error("sp_exact_plan: K >= 1 and output pointers required");
    return SP_ECONFIG;
  }
  int b = 0, n = 0;
  ozaki_plan(K, &b, &n);
  *bits = b;
  *nsl = n;
  return SP_OK;
}

int sp_exponents(int32_t axis, int64_t rows, int64_t cols, const double* X, int64_t ldx, int32_t* e, void* stream) {
  return axis == 1 ? row_exponents(rows, cols, X, ldx, e, ST(stream)) : col_exponents(rows, cols, X, ldx, e, ST(stream));
}

int sp_gemm_exact_levels(int32_t trans_a, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                         const int32_t* ea, const double* B, int64_t ldb, const int32_t* eb, int32_t bits,
                         int32_t nsl, double* levels, void* stream) {
  return gemm_exact_levels(trans_a, M, N, K, A, lda, ea, B, ldb, eb, bits, nsl, levels, ST(stream));
}

int sp_dd_levels(int64_t M, int64_t N, const double* levels, int32_t nsl, const double* tail, double* hi, double* lo,
                 int64_t ldc, void* stream) {
  return dd_levels(M, N, levels, nsl, tail, hi, lo, ldc, ST(stream));
}

int sp_pqd_begin(int64_t m, int64_t len, int32_t k, const double* E, int64_t lde, double* WK, int64_t* perm,
                 double* R, int64_t ldr, double* pn2, void* stream) {
  return pqd_begin(m, len, k, E, lde, WK, perm, R, ldr, pn2, ST(stream));
}

int sp_pqd_select(int32_t t, int32_t k, int64_t m, int64_t len, const double* n2, int64_t* perm, double* R,
                  int64_t ldr, double* WK, const double* Qt, double* delta, int64_t* jsel, void* stream) {
  return pqd_select(t, k, m, len, n2, perm, R, ldr, WK, Qt, delta, jsel, ST(stream));
}

int sp_pqd_orth(int32_t t, int64_t len, const double* delta, double* R, int64_t ldr, const double* WK, double* Qt,
                double* part2, void* stream) {
  return pqd_orth(t, len, delta, R, ldr, WK, Qt, part2, ST(stream));
}

int sp_pqd_coef(int32_t t, int64_t m, int64_t len, const double* p2, double* R, int64_t ldr, const double* WK,
                double* Qt, double* coef, int32_t* status, void* stream) {
  return pqd_coef(t, m, len, p2, R, ldr, WK, Qt, coef, status, ST(stream));
}

int sp_pqd_update(int32_t t, int64_t m, int64_t len, const double* coef, double* R, int64_t ldr, double* WK,
                  const double* Qt, double* pn2, void* stream) {
  return pqd_update(t, m, len, coef, R, ldr, WK, Qt, pn2, ST(stream));
}

int sp_id_from_qr(int64_t m, int32_t k, const int64_t* perm, const double* R, int64_t ldr, double* P,
                  int64_t* indices, int64_t* info, void* stream) {
  const int64_t l0 = launches();
  int warn = 0;
  const int st = id_from_qr(m, k, perm, R, ldr, P, indices, &warn, ST(stream));
  if (info) {
    for (int i = 0; i < SP_INFO_LEN; ++i) info[i] = 0;
    info[SP_INFO_WARN] = warn;
    info[SP_INFO_LAUNCHES] = launches() - l0;
  }
  return st;
}

int sp_tsqr(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq, double* R,
            int64_t ldr, void* stream) {
  return tsqr(rows, cols, X, ldx, Q, ldq, R, ldr, ST(stream));
}

int sp_qr_tall(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq, double* R,
               int64_t ldr, int32_t well_conditioned, void* stream) {
  return qr_tall(rows, cols, X, ldx, Q, ldq, R, ldr, well_conditioned != 0, ST(stream));
}

int sp_cholqr2_async(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq, double* R,
                     int64_t ldr, int32_t* dflag, void* stream) {
  return cholqr2_async(rows, cols, X, ldx, Q, ldq, R, ldr, dflag, ST(stream));
}

int sp_thin_qr(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
               double* R, int64_t ldr, void* stream) {
  return thin_qr(rows, cols, X, ldx, Q, ldq, R, ldr, ST(stream));
}

int sp_jacobi_svd(int64_t n, const double* M, int64_t ldm, double* U, int64_t ldu, double* S, double* V,
                  int64_t ldv, void* stream) {
  return jacobi_svd(n, M, ldm, U, ldu, S, V, ldv, ST(stream));
}

int sp_thin_svd(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* U, int64_t ldu,
                double* S, double* V, int64_t ldv, void* stream) {
  return thin_svd(rows, cols, X, ldx, U, ldu, S, V, ldv, ST(stream));
}

int sp_thin_svd_t(int64_t rows, int64_t cols, const double* Xt, int64_t ldxt, double* U, int64_t ldu, double* S,
                  double* V, int64_t ldv, void* stream) {
  return thin_svd_t(rows, cols, Xt, ldxt, U, ldu, S, V, ldv, ST(stream));
}

int sp_scale_columns(int64_t rows, int64_t cols, double* X, int64_t ldx, const double* d, int32_t divide,
                     void* stream) {
  return scale_columns(rows, cols, X, ldx, d, divide != 0, ST(stream));
}

int sp_gather_rows(const void* X, int32_t x_dtype, int64_t ldx, int64_t cols, const int64_t* idx, int64_t k,
                   double* out, int64_t ldo, void* stream) {
  return gather_rows(X, x_dtype, ldx, cols, idx, k, out, ldo, ST(stream));
}

int sp_fill_uniform(int64_t rows, int64_t cols, double* X, int64_t ldx, uint64_t seed, int64_t row_offset,
                    void* stream) {
  return fill_uniform(rows, cols, X, ldx, seed, ST(stream), row_offset);
}

int sp_pinv_apply(const double* s, int64_t count, double tol, double* out, void* stream) {
  return pinv_apply(s, count, tol, out, ST(stream));
}

int sp_trsm_upper(int64_t k, const double* R, int64_t ldr, int64_t ncols, const double* B, int64_t ldb,
                  double* X, int64_t ldx, void* stream) {
  return trsm_upper(k, R, ldr, ncols, B, ldb, X, ldx, ST(stream));
}

int sp_pivoted_qr(int64_t rows, int64_t cols, const double* Mt, int64_t ldmt, int32_t k, int64_t* perm,
                  double* Q, int64_t ldq, double* R, int64_t ldr, void* stream) {
  return pivoted_qr(rows, cols, Mt, ldmt, k, perm, Q, ldq, R, ldr, ST(stream));
}

int sp_row_id(int64_t m, int64_t cols, const double* M, int64_t ldm, int32_t k, double* P,
              int64_t* indices, int64_t* info, void* stream) {
  int warn = 0;
  const int64_t l0 = launches();
  const int st = row_id(m, cols, M, ldm, k, P, indices, &warn, ST(stream));
  if (info) {
    for (int i = 0; i < SP_INFO_LEN; ++i) info[i] = 0;
    info[SP_INFO_WARN] = warn;
    info[SP_INFO_LAUNCHES] = launches() - l0;
  }
  return st;
}

int sp_sketch_basis(const double* X, int64_t rows, int64_t cols, int64_t ldx, double power, int32_t r_max,
                    double* U, int64_t ldu, double* S, int64_t* info, void* stream) {
  return sketch_basis(X, rows, cols, ldx, power, r_max, U, ldu, S, info, ST(stream));
}

int sp_srht_sketch(int64_t rows, int64_t cols, const double* X, int64_t ldx, int32_t b, uint64_t seed,
                   double* Y, int64_t ldy, int32_t* flag, void* stream) {
  return srht_sketch(rows, cols, X, ldx, b, seed, Y, ldy, flag, ST(stream));
}

int sp_gram_chol_dd(int64_t rows, int32_t b, const double* X, int64_t ldx, double* R, int64_t ldr, void* stream) {
  Arena ar(ST(stream));
  return gram_chol_dd(rows, b, X, ldx, R, ldr, ar, ST(stream));
}

int sp_srht_gather(const void* A, int32_t a_dtype, int64_t rows, int64_t lda, const int64_t* gidx, int64_t cols,
                   double* X, int64_t ldx, int32_t b, uint64_t seed, double* Y, int64_t ldy, int32_t* flag,
                   void* stream) {
  if (a_dtype != SP_F64 && a_dtype != SP_F32) {
    set_error("unknown dtype tag");
    return SP_ECONFIG;
  }
  return srht_gather(A, a_dtype, rows, lda, gidx, cols, X, ldx, b, seed, Y, ldy, flag, ST(stream));
}

int sp_householder_complete(int64_t N, int32_t r, int32_t k, double* out, int64_t ldo, double* kp_out,
                            void* stream) {
  return householder_complete(N, r, k, out, ldo, ST(stream), kp_out);
}

int sp_single_pass_svd(const void* A, int32_t a_dtype, int64_t m, int64_t n, int64_t lda,
                       const int64_t* idx, const double* w, int32_t depth, int64_t n_c,
                       const double* omega, int64_t ell, int32_t k, const double* pre_s0, double* U,
                       double* S, double* V, int64_t* info, void* stream) {
  return single_pass_svd(A, a_dtype, m, n, lda, idx, w, depth, n_c, omega, ell, k, pre_s0, U, S, V, info,
                         ST(stream));
}

int sp_power_svd(const void* A, int32_t a_dtype, int64_t m, int64_t n, int64_t lda, const int64_t* idx,
                 const double* w, int32_t depth, int64_t n_c, const double* omega, int64_t ell,
                 const int64_t* cols, int64_t n_cols, int32_t q, int32_t k, const double* pre_s0,
                 const double* pre_c, int32_t hints, double* U, double* S, double* V, int64_t* info,
                 void* stream) {
  return power_svd(A, a_dtype, m, n, lda, idx, w, depth, n_c, omega, ell, cols, n_cols, q, k, pre_s0, pre_c,
                   hints, U, S, V, info, ST(stream));
}

int sp_power_id(const void* A, int32_t a_dtype, int64_t m, int64_t n, int64_t lda, const int64_t* idx,
                const double* w, int32_t depth, int64_t n_c, const int64_t* cols, int64_t n_cols, int32_t q,
                int32_t k, int32_t r_req, const double* project_omega, int64_t project_ell,
                int32_t id_on_basis, const double* pre_s0, const double* pre_c, double* P,
                int64_t* indices, double* skeleton, double* lift_left, double* lift_right, double* lift_ur,
                int32_t r_max, int64_t* info, void* stream) {
  return power_id(A, a_dtype, m, n, lda, idx, w, depth, n_c, cols, n_cols, q, k, r_req, project_omega,
                  project_ell, id_on_basis, pre_s0, pre_c, P, indices, skeleton, lift_left, lift_right, lift_ur,
                  r_max, info, ST(stream));
}

int sp_frob_residual(const void* A, int32_t a_dtype, int64_t m, int64_t n, int64_t lda, const double* U,
                     int64_t ldu, const double* S, const double* V, int64_t ldv, int32_t k, double* out2,
                     void* stream) {
  return frob_residual(A, a_dtype, m, n, lda, U, ldu, S, V, ldv, k, out2, ST(stream));
}

}  // extern "C"
