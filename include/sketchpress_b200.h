/*
 * sketchpress_b200.h -- C-ABI of the B200-native single-pass sketch compressor.
 *
 * Drop-in boundary for the hot path of the reference package `sketchpress`
 * (arXiv 2105.01271; reference sources under pkg/src/sketchpress/, cited as
 * src/<file>:<line>).  The reference is pure Python with no FFI layer, so each
 * entry point below replaces one reference Python function (named in its
 * comment); the Python host mirror (paper_2105_01271_b200/) binds them with
 * ctypes exactly as a maintainer would bind them from the reference
 * (INTEGRATION.md shows that stub).
 *
 * Conventions
 *   - All matrices are ROW-MAJOR with an explicit leading dimension counted in
 *     elements.  All pointers are DEVICE pointers unless marked (host).
 *   - `stream` is a cudaStream_t passed as void*; every call is stream-ordered
 *     and asynchronous unless it says it synchronises (the pipelines do, to
 *     read the kept rank).
 *   - `a_dtype` tags the snapshot matrix A: SP_F64 or SP_F32 (FP32-stored A is
 *     widened to FP64 on load, the semantics of src/snapshot_io.py:171).
 *   - Return value: a status (0 ok, 2 config, 3 I/O, 4 numerical -- the CLI
 *     exit codes of src/cli.py:28-30 -- plus 5 for CUDA failures).  The message
 *     of the last failure on the calling thread is sp_last_error().
 *   - Warnings (src/errors.py:28 RankDeficiencyWarning) come back as bits in
 *     an `info` array (SP_WARN_*), which the host mirror turns into Python
 *     warnings.
 */
#ifndef SKETCHPRESS_B200_H
#define SKETCHPRESS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_ABI_VERSION 1

/* status codes */
#define SP_OK 0
#define SP_ECONFIG 2     /* ConfigError (src/errors.py:8)        */
#define SP_EIO 3         /* FormatError / StreamPoisonedError     */
#define SP_ENUMERICAL 4  /* NumericalError (src/errors.py:24)     */
#define SP_ECUDA 5       /* CUDA runtime / launch failure         */

/* dtype tags for A */
#define SP_F64 0
#define SP_F32 1

/* warning bits returned in info[SP_INFO_WARN] */
#define SP_WARN_RANK_DEFICIENT 1 /* regularized (pinv) solve taken        */
#define SP_WARN_LIFT_CLAMPED 2   /* lifting rank clamped to sketch rank   */
#define SP_WARN_ID_PINV 4        /* row_id pseudo-inverse fallback        */
#define SP_WARN_BULK_SPLIT 8     /* device diagnostic (no reference warning): the ID lifting
                                    rank r splits a flat stretch of the sketch spectrum wider
                                    than the exact-SVD limit; its rank-r subspace is resolved
                                    only above that stretch  */

/* layout of the host `info` array filled by the pipelines (length SP_INFO_LEN) */
#define SP_INFO_KEPT 0      /* effective rank of the projector (r_kept)      */
#define SP_INFO_WARN 1      /* SP_WARN_* bits                                 */
#define SP_INFO_BLOCK 2     /* range-finder block width used                  */
#define SP_INFO_ITERS 3     /* range-finder subspace iterations               */
#define SP_INFO_RANK 4      /* ID: numerical rank of the coarse sketch (>=)   */
#define SP_INFO_LIFT_R 5    /* ID: lifting rank actually used                 */
#define SP_INFO_LAUNCHES 6  /* device kernels launched by the call            */
#define SP_INFO_FUSED 7     /* 1: this call took the fused (deferred-status) finish:
                               its breakdown / non-finite flag is read with
                               sp_deferred_status after the caller's sync     */
#define SP_INFO_LEN 8

int sp_abi_version(void);
const char* sp_last_error(void);
/* Number of kernels this library launched on the calling thread so far. */
int64_t sp_launch_count(void);
/* Hand every cached workspace block of the current device back to the CUDA
 * memory pool and trim the pool (synchronises the device).  The library keeps
 * its workspaces across calls (stream-ordered free lists: no allocation on
 * the critical path of a call); a host application calls this when it wants
 * the HBM back, e.g. between problems of very different size.  Blocks of every
 * size are kept, up to 64 GB per device (environment: SPB_WS_CACHE_CAP_GB,
 * SPB_WS_CACHE_MAX_MB = largest kept block); an allocation failure inside the
 * library drains them and retries once.  No reference counterpart (numpy frees
 * its temporaries itself).
 */
int sp_release_workspaces(void);

/* Deferred status of the calling thread's last pipeline call: the fused
 * finish stage (r <= 16 kept columns, kappa < 1e6) runs without a host
 * synchronisation and raises a device flag on a Cholesky breakdown or
 * non-finite data (S is then NaN).  Waits for that call's completion and
 * returns the flag in *flag (0 = clean).  The reference raises at the same
 * point synchronously (NumericalError, src/kernels.py:47-49); the Python
 * mirror reads this after its device->host copies and re-runs the call with
 * sp_set_finish_mode(1) (Householder TSQR finish). */
int sp_deferred_status(int32_t* flag);
/* 0 = automatic (fused CholeskyQR2 finish when it applies), 1 = Householder
 * TSQR finish (thread-local). */
int sp_set_finish_mode(int32_t mode);

/* ---------------------------------------------------------------- K1 -----
 * out[i, c] = sum_t A[i, idx[t, c]] * w[t, c]      (t = 0..depth-1, no FMA)
 * Replaces apply_sketch for the stencil kinds (src/sketch.py:171-184,
 * loop at :179-181) and, with exact_copy=1 (depth must be 1, w ignored),
 * gather_columns (src/sketch.py:201-211).  idx / w are (depth x n_c)
 * row-major (the SketchOperator tables, src/sketch.py:161-168).  Bit-exact
 * with the reference: the product and the running sum are each rounded.
 */
int sp_apply_stencil(const void* A, int32_t a_dtype, int64_t rows, int64_t n, int64_t lda,
                     const int64_t* idx, const double* w, int32_t depth, int64_t n_c,
                     int32_t exact_copy, double* out, int64_t ldo, void* stream);

/* Validation of a column index set (src/sketch.py:206-210 / src/power.py:216-224):
 * returns SP_ECONFIG if empty, out of [0, n) or not distinct.  Synchronises. */
int sp_check_columns(const int64_t* cols, int64_t count, int64_t n, void* stream);

/* ---------------------------------------------------------------- K2 -----
 * Y (n x r) = A^T Z,  A (m x n), Z (m x r).  The single read of A that
 * replaces the per-block `gram += block.T @ out` / `hc += block.T @ sub`
 * products (src/svd.py:66, src/power.py:209-211) in the reformulated
 * single-pass algebra.  FP64 accumulation, fixed reduction
 * order (bitwise reproducible).  Any r >= 1 (r > 16 routes to the DMMA GEMM).
 */
int sp_skinny_atz(const void* A, int32_t a_dtype, int64_t m, int64_t n, int64_t lda,
                  const double* Z, int64_t ldz, int32_t r, double* Y, int64_t ldy,
                  void* stream);

/* ---------------------------------------------------------------- K3 -----
 * C = alpha * op(A) op(B) + beta * C, FP64 on the DMMA tensor pipe
 * (mma.sync.m8n8k4.f64).  op(X) = X (trans=0) or X^T (trans=1).  op(A) is
 * M x K, op(B) is K x N.  Replaces every numpy `@` on the path (e.g.
 * src/power.py:101,105,166-170,284; src/rowid.py:138-139) and the literal
 * cross-Gramian H = A^T (A D) (src/svd.py:66).  Deterministic split-K.
 */
int sp_gemm(int32_t trans_a, int32_t trans_b, int64_t M, int64_t N, int64_t K, double alpha,
            const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
            double* C, int64_t ldc, void* stream);

/* W = A A^T (M x M, A row-major M x K): the symmetric product of the power
 * enrichment in its (C C^T) s0 association (src/power.py:99-108, 282-285; used
 * when the column set is wider than the snapshot count, cfg5).  Only the
 * tiles on and above the diagonal are computed, the rest is mirrored: W is
 * exactly symmetric at half the DMMA work of sp_gemm(0, 1, ...).
 */
int sp_gemm_aat(int64_t M, int64_t K, const double* A, int64_t lda, double* W, int64_t ldw,
                void* stream);

/* --------------------------------------------------------------- K3x -----
 * C_hi (+ C_lo) = op(A) (B_hi + B_lo), nearly exactly rounded: Ozaki slices of
 * A's rows and B's columns, every level sum an exact DMMA GEMM, levels summed
 * in double-double (error below ~2^-56 of sum_l |a_il||b_lj|).  op(A) = A
 * (trans_a = 0, M x K) or A^T (A is K x M); B is K x N; B_lo and C_lo may be
 * NULL.  The enrichment E = C (C^T s0) of power_id (src/power.py:282-285),
 * whose greedy pivots are decided by ulp-level residual differences.
 */
int sp_gemm_exact(int32_t trans_a, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                  const double* B_hi, const double* B_lo, int64_t ldb, double* C_hi, double* C_lo,
                  int64_t ldc, void* stream);

/* Building blocks of sp_gemm_exact for operands split across ranks (the
 * sharded ID's W = sum_i C_i C_i^T): the slice plan for a total depth K, the
 * per-row (axis = 1) / per-column (axis = 0) max exponents (allreduce-max them
 * across ranks so every rank slices on the same grid), the nsl exact level
 * products (levels: nsl x M x N; exact for any summation order, so their
 * allreduce-sum is exact) and their double-double sum (+ an inexact tail). */
int sp_exact_plan(int64_t K, int32_t* bits, int32_t* nsl);
int sp_exponents(int32_t axis, int64_t rows, int64_t cols, const double* X, int64_t ldx, int32_t* e, void* stream);
int sp_gemm_exact_levels(int32_t trans_a, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                         const int32_t* ea, const double* B, int64_t ldb, const int32_t* eb, int32_t bits,
                         int32_t nsl, double* levels, void* stream);
int sp_dd_levels(int64_t M, int64_t N, const double* levels, int32_t nsl, const double* tail, double* hi,
                 double* lo, int64_t ldc, void* stream);

/* ---------------------------------------------------------------- K4 -----
 * Householder QR of a tall matrix X (rows x cols, rows >= cols): explicit
 * Q (rows x cols) and R (cols x cols).  cols <= 32 runs as a register-resident
 * TSQR tree; wider inputs are processed in 32-column panels with two passes
 * of block Gram-Schmidt between them.  Q, R may not alias X.
 */
int sp_tsqr(int64_t rows, int64_t cols, const double* X, int64_t ldx,
            double* Q, int64_t ldq, double* R, int64_t ldr, void* stream);

/* Tall QR with a conditioning hint: well_conditioned != 0 (caller certifies
 * kappa(X) < ~1e6, cols <= 112) runs CholeskyQR2 (Gram + Cholesky on the DMMA
 * GEMM, two passes), falling back to Householder TSQR on breakdown;
 * otherwise Householder TSQR.  Synchronises once on the CholeskyQR2 path. */
int sp_qr_tall(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
               double* R, int64_t ldr, int32_t well_conditioned, void* stream);

/* CholeskyQR2 without a host synchronisation: a Cholesky breakdown ORs 1
 * into the device int *dflag (caller zeroes it and reads it later, redoing
 * the factorisation with sp_tsqr if it is set).  cols <= 112. */
int sp_cholqr2_async(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* Q, int64_t ldq,
                     double* R, int64_t ldr, int32_t* dflag, void* stream);

/* thin_qr (src/kernels.py:74-84): reduced QR of any rows x cols matrix with
 * the reference sign convention (src/kernels.py:52-71).  Q is rows x p,
 * R is p x cols with p = min(rows, cols).  Requires p <= 256. */
int sp_thin_qr(int64_t rows, int64_t cols, const double* X, int64_t ldx,
               double* Q, int64_t ldq, double* R, int64_t ldr, void* stream);

/* ---------------------------------------------------------------- K5 -----
 * One-sided (Hestenes) Jacobi SVD of a square n x n matrix in one CTA:
 * M = U diag(S) V^T, S descending.  n <= 256.  Columns of U whose singular
 * value is exactly zero are returned as zero vectors. */
int sp_jacobi_svd(int64_t n, const double* M, int64_t ldm, double* U, int64_t ldu,
                  double* S, double* V, int64_t ldv, void* stream);

/* thin_svd (src/kernels.py:87-94): U (rows x p), S (p), V (cols x p),
 * p = min(rows, cols) <= 256, reference sign convention on U with V. */
int sp_thin_svd(int64_t rows, int64_t cols, const double* X, int64_t ldx,
                double* U, int64_t ldu, double* S, double* V, int64_t ldv, void* stream);

/* thin_svd of X (rows x cols, rows <= cols) given Xt = X^T (cols x rows,
 * ld ldxt) without transposing: the projected matrix of the two-pass SVDs
 * (src/svd.py:137-143, src/power.py:143-156) arrives from the A pass as
 * (Q^T A)^T = A^T Q.  Same outputs and sign convention as sp_thin_svd. */
int sp_thin_svd_t(int64_t rows, int64_t cols, const double* Xt, int64_t ldxt,
                  double* U, int64_t ldu, double* S, double* V, int64_t ldv, void* stream);

/* X[:, j] /= d[j] (divide != 0, the `vt /= s_k` of direct_svd,
 * src/svd.py:113) or X[:, j] *= d[j]. */
int sp_scale_columns(int64_t rows, int64_t cols, double* X, int64_t ldx, const double* d,
                     int32_t divide, void* stream);

/* out[i, :] = X[idx[i], :] for i < k (X f64 or f32, widened to f64): the
 * fine skeleton rows of the two-pass IDs (_gather_rows, src/rowid.py:82-95). */
int sp_gather_rows(const void* X, int32_t x_dtype, int64_t ldx, int64_t cols,
                   const int64_t* idx, int64_t k, double* out, int64_t ldo, void* stream);

/* X (rows x cols, ld ldx) = rows [row_offset, row_offset + rows) of the
 * seed's uniform(-1, 1) test block (counter-based hash of the global index
 * row * cols + col): the random range-finder block of the sketch basis, so
 * a rank owning a slab of the coarse columns generates exactly its rows
 * (column-sharded power_svd). */
int sp_fill_uniform(int64_t rows, int64_t cols, double* X, int64_t ldx, uint64_t seed,
                    int64_t row_offset, void* stream);

/* ---------------------------------------------------------------- K6 -----
 * pinv_apply (src/kernels.py:158-168): out = 1/s where s > tol * s[0], else 0. */
int sp_pinv_apply(const double* s, int64_t count, double tol, double* out, void* stream);

/* X = R^{-1} B for upper-triangular R (k x k): the solve_triangular(r1, r2)
 * of row_id (src/rowid.py:68).  B, X are k x ncols. */
int sp_trsm_upper(int64_t k, const double* R, int64_t ldr, int64_t ncols,
                  const double* B, int64_t ldb, double* X, int64_t ldx, void* stream);

/* ---------------------------------------------------------------- K7 -----
 * pivoted_qr (src/kernels.py:97-142) of M (rows x cols), supplied as
 * Mt = M^T (cols x rows row-major, i.e. M column-major) so every candidate
 * column is contiguous.  Greedy max residual norm, exact ties to the lowest
 * original index, one re-orthogonalisation, zero-pivot filler, final sign
 * convention.  Outputs: perm (cols, int64), Q (rows x k), R (k x cols).
 * Mt is not modified. */
int sp_pivoted_qr(int64_t rows, int64_t cols, const double* Mt, int64_t ldmt, int32_t k,
                  int64_t* perm, double* Q, int64_t ldq, double* R, int64_t ldr,
                  void* stream);

/* row_id (src/rowid.py:53-79) of M (m x cols): pivoted_qr(M^T, k), then
 * C = R1^{-1} R2 (triangular solve, or the pseudo-inverse fallback with
 * SP_WARN_ID_PINV), P (m x k) with P[indices] = I exactly, indices (k). */
int sp_row_id(int64_t m, int64_t cols, const double* M, int64_t ldm, int32_t k, double* P,
              int64_t* indices, int64_t* info, void* stream);

/* ------------------------------------------------- K7 across ranks -----
 * The greedy pivoted QR of src/kernels.py:97-142 on candidates (rows of the
 * enriched sketch E, m of them) whose entries are sharded over ranks: this
 * rank holds E_i (m x len, candidate j = row j).  Per step t the caller
 * allreduce-sums the partial outputs between the calls:
 *   sp_pqd_begin  -> pn2 (m)      partial ||w_j||^2          (before step 0)
 *   sp_pqd_select(n2 = sum pn2)  -> delta (t) partial Q^T w_t; pivot, swaps
 *   sp_pqd_orth  (delta summed)   -> part2 (1) partial ||v||^2
 *   sp_pqd_coef  (part2 summed)   -> coef (m) partial v . w_j
 *   sp_pqd_update(coef summed)    -> pn2 (m) for the next step
 * perm (m) and R (k x m, ld ldr) come out identical on every rank; WK (m x len),
 * Qt (k x len) are this rank's work rows; jsel (1), status (1, zero it first:
 * SP_ENUMERICAL on an exactly zero pivot) device words. */
int sp_pqd_begin(int64_t m, int64_t len, int32_t k, const double* E, int64_t lde, double* WK, int64_t* perm,
                 double* R, int64_t ldr, double* pn2, void* stream);
int sp_pqd_select(int32_t t, int32_t k, int64_t m, int64_t len, const double* n2, int64_t* perm, double* R,
                  int64_t ldr, double* WK, const double* Qt, double* delta, int64_t* jsel, void* stream);
int sp_pqd_orth(int32_t t, int64_t len, const double* delta, double* R, int64_t ldr, const double* WK, double* Qt,
                double* part2, void* stream);
int sp_pqd_coef(int32_t t, int64_t m, int64_t len, const double* p2, double* R, int64_t ldr, const double* WK,
                double* Qt, double* coef, int32_t* status, void* stream);
int sp_pqd_update(int32_t t, int64_t m, int64_t len, const double* coef, double* R, int64_t ldr, double* WK,
                  const double* Qt, double* pn2, void* stream);

/* The interpolation coefficients of row_id (src/rowid.py:53-79) from a
 * pivoted QR of M^T: C = R1^-1 R2 (pseudo-inverse solve, SP_WARN_ID_PINV,
 * when R1 is rank deficient); P (m x k) with P[perm[:k]] = I and
 * P[perm[k:]] = C^T; indices = perm[:k]. */
int sp_id_from_qr(int64_t m, int32_t k, const int64_t* perm, const double* R, int64_t ldr, double* P,
                  int64_t* indices, int64_t* info, void* stream);

/* Kept left basis of a sketch X (rows x cols): the top singular triplets by
 * randomized block subspace iteration (Householder TSQR + Jacobi Rayleigh-
 * Ritz; exact TSQR + Jacobi when min(rows, cols) <= 64) and the reference's
 * kept-rank rule r = #{(s_i/s_1)^power > 1e-12} (src/kernels.py:19, 158-168;
 * power = 2q+1 for the power pipeline's G = (C C^T)^q C).  Writes U (rows x
 * min(r, r_max), ld ldu) and S; info[SP_INFO_KEPT] = r.  Used by the
 * column-sharded driver on the all-gathered C.  Synchronises. */
int sp_sketch_basis(const double* X, int64_t rows, int64_t cols, int64_t ldx, double power, int32_t r_max,
                    double* U, int64_t ldu, double* S, int64_t* info, void* stream);

/* R factor of a tall block X (rows x b, b <= 32, rows >= b) with
 * R^T R = X^T X, from the Gram accumulated and Cholesky-factored in
 * double-double arithmetic (ddgram.cu); pivots below 1e-29 trace(X^T X) give
 * zero rows.  Replaces thin_qr's R (src/kernels.py:62-84) for the
 * Rayleigh-Ritz core of the sketch-side subspace iteration, which needs R
 * only.  R is b x b row-major (ld ldr), zero below the diagonal.  Asynchronous. */
int sp_gram_chol_dd(int64_t rows, int32_t b, const double* X, int64_t ldx, double* R, int64_t ldr, void* stream);

/* Range-finder test block of the sketch-side subspace iteration (srht.cu):
 * Y (rows x b, ld ldy) = X D H S -- random signs, Walsh-Hadamard transform of
 * the zero-padded width, b stratified column samples (the structured
 * replacement of the dense Gaussian block of np.random-style range finders;
 * Halko, Martinsson & Tropp sec. 4.6).  cols <= 16384, b <= 32.  *flag
 * (device int, may be NULL) is OR-ed with 1 if X has a non-finite entry.
 * sp_srht_gather forms X = A(:, gidx) (exact copies, written to X) and the
 * same Y in one pass over A (K1 fused with the first product; the power
 * pipeline uses it for a device-resident A); wider than 16384 columns, the
 * row is cut into 16384-column chunks with their own signs and the same
 * samples, and the chunk transforms are summed in chunk order (a block SRHT:
 * Omega^T Omega = chunks * 16384 * I).  SP_ECONFIG outside the range. */
int sp_srht_sketch(int64_t rows, int64_t cols, const double* X, int64_t ldx, int32_t b, uint64_t seed,
                   double* Y, int64_t ldy, int32_t* flag, void* stream);
int sp_srht_gather(const void* A, int32_t a_dtype, int64_t rows, int64_t lda, const int64_t* gidx, int64_t cols,
                   double* X, int64_t ldx, int32_t b, uint64_t seed, double* Y, int64_t ldy, int32_t* flag,
                   void* stream);

/* Orthonormal completion of out[:, 0:r) (orthonormal, N x r) into
 * out[:, r:k) by Householder reconstruction (LU of Q - [S;0]; no QR).  If
 * kp_out (r x (k-r)) is non-NULL it receives K', so that for a row-sharded Q
 * every other row block i of the completion is -Q_i K' (the rows 0..k-1 live
 * in the block this call factors).  Requires r <= 32, k <= 256, N >= k. */
int sp_householder_complete(int64_t N, int32_t r, int32_t k, double* out, int64_t ldo, double* kp_out,
                            void* stream);

/* ------------------------------------------------------- pipelines -----
 * Device-resident single-pass pipelines.  A is m x n (lda), the sketch is
 * the stencil table (idx, w: depth x n_c) optionally composed with a dense
 * Gaussian projection omega (n_c x ell, device, or NULL), and `cols` is the
 * power-iteration column set I (src/power.py:64-67).  Inputs are validated
 * like the reference (ConfigError) before any kernel runs.  Outputs are
 * row-major device buffers:  U (m x k), S (k), V (n x k).  `info` (host,
 * SP_INFO_LEN int64) receives the kept rank, warning bits and counters.
 *
 * If `pre_s0` (m x out_dim) / `pre_c` (m x n_cols) are non-NULL they hold the
 * sketch / column block already gathered while A was ingested (the fused
 * ingest path of the host streams), and the gather is skipped.
 */

/* single_pass_svd (src/svd.py:168-189). */
int sp_single_pass_svd(const void* A, int32_t a_dtype, int64_t m, int64_t n, int64_t lda,
                       const int64_t* idx, const double* w, int32_t depth, int64_t n_c,
                       const double* omega, int64_t ell, int32_t k,
                       const double* pre_s0,
                       double* U, double* S, double* V, int64_t* info, void* stream);

/* hints for sp_power_svd (0 = verify everything on the device) */
#define SP_HINT_COLS_VALIDATED 1 /* caller checked I: in [0, n) and distinct   */
#define SP_HINT_SAME_SET 2       /* caller asserts s0 == A(:, I) (unit injection on I, no projection) */
#define SP_HINT_DIFFERENT_SET 4  /* caller asserts s0 != A(:, I)               */

/* power_svd, single_pass mode (src/power.py:227-249, 124-181). */
int sp_power_svd(const void* A, int32_t a_dtype, int64_t m, int64_t n, int64_t lda,
                 const int64_t* idx, const double* w, int32_t depth, int64_t n_c,
                 const double* omega, int64_t ell,
                 const int64_t* cols, int64_t n_cols, int32_t q, int32_t k,
                 const double* pre_s0, const double* pre_c, int32_t hints,
                 double* U, double* S, double* V, int64_t* info, void* stream);

/* power_id, single_pass mode (src/power.py:252-308) and single_pass_id
 * (src/rowid.py:142-183, with q = 0 and cols = NULL).  The lifting
 * operator T = V_r S_r^{-1} U_r^T A (src/rowid.py:115-139) is returned
 * FACTORED: lift_left = V_r S_r^{-1} (n_c x r_max, ld r_max) and, when
 * non-NULL, lift_right = U_r^T A (r_max x n, ld n) and/or lift_ur = U_r
 * (m x r_max, ld r_max) -- the right factor can stay implicit (U_r with A)
 * when r x n does not fit beside A.  The used rank is info[SP_INFO_LIFT_R];
 * r_max is the caller's buffer width (>= the requested / default r).
 * project_omega (n_c x project_ell) narrows the selection input; id_on_basis
 * selects on the leading k left singular vectors of the sketch instead.
 * Outputs: P (m x k), indices (k, int64), skeleton (k x n_c).  r_req <= 0
 * means the reference default max(k, min(2k, rank)). */
int sp_power_id(const void* A, int32_t a_dtype, int64_t m, int64_t n, int64_t lda,
                const int64_t* idx, const double* w, int32_t depth, int64_t n_c,
                const int64_t* cols, int64_t n_cols, int32_t q, int32_t k, int32_t r_req,
                const double* project_omega, int64_t project_ell, int32_t id_on_basis,
                const double* pre_s0, const double* pre_c,
                double* P, int64_t* indices, double* skeleton,
                double* lift_left, double* lift_right, double* lift_ur, int32_t r_max,
                int64_t* info, void* stream);

/* ---------------------------------------------------------------- K8 -----
 * ||A - U diag(S) V^T||_F^2 and ||A||_F^2 streamed over A (never forming the
 * m x n product): the rel_frob_error metric (src/analysis.py:57-65) of a
 * LowRankSVD.reconstruct() (src/svd.py:42-43) and of the CLI --verify pass
 * (src/cli.py:125-139, left (m x k) . right (k x n) with S = 1, V = right^T).
 * k <= 256.  out2 (host) = {err2, ref2}.  Synchronises. */
int sp_frob_residual(const void* A, int32_t a_dtype, int64_t m, int64_t n, int64_t lda,
                     const double* U, int64_t ldu, const double* S, const double* V,
                     int64_t ldv, int32_t k, double* out2, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SKETCHPRESS_B200_H */
