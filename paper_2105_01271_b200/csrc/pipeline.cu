// Device-resident single-pass pipelines: single_pass_svd, power_svd (single
// pass) and power_id / single_pass_id.  Host-side C++ orchestration of the
// K1..K7 kernels; the only host synchronisations are the reads of the small
// Ritz spectra that fix the kept rank (and the finite checks the reference
// performs).
//
// Algebra:  the reference returns
// the rank-k SVD of P_r A, where P_r projects onto the top r left singular
// vectors of G = (C C^T)^q s0 and r = #{sigma_i(G) > 1e-12 sigma_1(G)} (the
// pinv cut of src/svd.py:159-165 / src/power.py:175-180; r = l on the
// triangular-solve branch).  We compute U_G from the sketch, then make ONE
// read of A for Y = A^T U_{G,r} (K2), then TSQR + Jacobi of the r x r core:
//   P_r A = U_r Y^T = U_r R_Y^T Q_Y^T = (U_r u~) s (Q_Y v~)^T.
// When s0 and C are the same column set (every BASELINE configuration),
// sigma(G) = sigma(C)^(2q+1) and U_G = U_C, so G is never formed and the kept
// basis is accurate to ~1e-16 sigma_1 instead of ~1e-16 sigma_1(G).
#include <atomic>
#include <map>
#include <mutex>
#include <cmath>
#include <cstring>
#include <vector>

#include <cstdlib>

#include "common.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace spb {

constexpr double kRankTol = 1e-12;  // src/kernels.py:19

int srht_sketch(int64_t rows, int64_t cols, const double* X, int64_t ldx, int b, uint64_t seed, double* Y,
                int64_t ldy, int* flag, cudaStream_t s);
bool srht_ok(int64_t rows, int64_t cols, int b);
bool srht_gather_ok(int64_t rows, int64_t cols, int b);
int srht_gather(const void* A, int a_dtype, int64_t rows, int64_t lda, const int64_t* gidx, int64_t cols, double* C,
                int64_t ldc, int b, uint64_t seed, double* Y, int64_t ldy, int* flag, cudaStream_t s);
constexpr uint64_t kSrhtSeed = 0x5eed5eedull;  // + block width

static int count_kept(const std::vector<double>& s, double power) {
  if (s.empty() || !(s[0] > 0.0)) return 0;
  int c = 0;
  for (double x : s)
    if (std::pow(x / s[0], power) > kRankTol) ++c;
  return c;
}

// exact SVD fallback of svd_top's ID mode up to this many columns: the
// size-general thin_svd (BCGS2 TSQR + block Jacobi) of the whole sketch
// (1.6 s at 5000 x 4096, cfg3: every block-Jacobi round streams W and V
// from HBM); wider flat stretches are resolved only above the stretch and
// flagged
constexpr int64_t kExactMax = 2048;
// ... and only while the sketch's long side keeps the panel TSQR cheap: cfg5's
// 2000 x 262144 FP32-floor sketch costs 1.8 s exact (BCGS2 over 262144 rows
// + the 2000-wide block Jacobi) against 0.9 s resolved above the floor
constexpr int64_t kExactLong = 16384;

struct TopSvd {
  int b = 0, kept = 0, iters = 0;
  bool bulk = false;  // ID mode: the leading `need` triplets split an unresolvable flat stretch
  double* U = nullptr;  // rows x b
  double* S = nullptr;  // b
  double* V = nullptr;  // cols x b
  std::vector<double> hs;
};

// Top singular triplets of X (rows x cols).  Exact (TSQR + Jacobi) when
// min(rows, cols) <= 64; otherwise a randomized block subspace iteration
// with Householder orthogonalisation and a Rayleigh-Ritz Jacobi step,
// iterated until the kept Ritz values are stable, growing the block when the
// kept rank gets within 8 of its width.
// `pflag` (device int, may be null) is a pending non-finite flag for X raised
// by an earlier asynchronous check; it is read with the first Ritz spectrum
// (no extra synchronisation) and turns into SP_ENUMERICAL with `pmsg`.
// check_input: svd_top raises the flag itself when X has a non-finite entry,
// detected on its first product Y = X Omega (Omega has no zero entries, so a
// non-finite X always yields a non-finite Y): an m x b check instead of a
// full pass over X.
struct PendingFlag {
  int* dev = nullptr;
  const char* msg = "";
  bool check_input = false;
};

static int read_flag_with(const PendingFlag& pf, int& host_flag, PinnedReads& rd) {
  host_flag = 0;
  if (pf.dev) SPB_TRY(rd.add(&host_flag, pf.dev, sizeof(int)));
  return SP_OK;
}

// -------------------------------------------------------------- doorbell ----
// Low-latency publication of a small device result (a Ritz spectrum and a
// pending flag) to the host: a one-CTA kernel copies it into mapped pinned
// memory and then bumps a sequence word, on which the host spins.  Replaces
// a device->host copy + stream synchronisation (copy-engine and wake-up
// latency) on the one host decision of the pipeline, the kept rank.
struct Doorbell {
  unsigned char* h = nullptr;  // [seq (u32) | flag (i32) | pad | values (f64)]
  unsigned next = 0;
};
static thread_local Doorbell t_bell;
constexpr int kBellMax = 1024;  // doubles

__global__ void publish_kernel(const double* __restrict__ v, int nv, const int* __restrict__ flag,
                               unsigned char* __restrict__ bell, unsigned seq, double* __restrict__ vcopy) {
  SPB_PDL_ENTRY();
  double* hv = reinterpret_cast<double*>(bell + 16);
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    hv[i] = v[i];
    if (vcopy) vcopy[i] = v[i];  // device copy of the spectrum (no memcpy node in the chain)
  }
  if (threadIdx.x == 0) *reinterpret_cast<volatile int*>(bell + 4) = flag ? *flag : 0;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) *reinterpret_cast<volatile unsigned*>(bell) = seq;
}

// enqueue the publication of v[0:nv) (+ *flag) on s; returns the sequence number
static int bell_publish(const double* v, int nv, const int* flag, unsigned& seq, cudaStream_t s,
                        double* vcopy = nullptr) {
  if (nv > kBellMax) {
    set_error("doorbell payload too large");
    return SP_ECUDA;
  }
  if (!t_bell.h) {
    void* p = nullptr;
    SPB_CUDA(cudaHostAlloc(&p, 16 + kBellMax * sizeof(double), cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(p, 0, 16);
    t_bell.h = static_cast<unsigned char*>(p);
  }
  seq = ++t_bell.next;
  if (seq == 0) seq = ++t_bell.next;
  unsigned char* d = nullptr;
  SPB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), t_bell.h, 0));
  SPB_CUDA(launch_pdl((publish_kernel), dim3(1), dim3(128), 0, s, v, nv, flag, d, seq, vcopy));
  count_launch();
  SPB_CHECK_LAUNCH();
  return SP_OK;
}

// spin until the publication `seq` has landed; copy it out
static int bell_wait(unsigned seq, double* v, int nv, int* flag, cudaStream_t s) {
  volatile unsigned* sq = reinterpret_cast<volatile unsigned*>(t_bell.h);
  for (unsigned it = 1;; ++it) {
    if (*sq == seq) break;
    if ((it & 4095) == 0) {  // the stream failed or drained without publishing
      const cudaError_t e = cudaStreamQuery(s);
      if (e == cudaSuccess && *sq != seq) {
        set_error("doorbell: stream idle without publication");
        return SP_ECUDA;
      }
      if (e != cudaSuccess && e != cudaErrorNotReady) {
        set_error(std::string("doorbell: ") + cudaGetErrorString(e));
        return SP_ECUDA;
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  if (flag) *flag = *reinterpret_cast<volatile int*>(t_bell.h + 4);
  if (nv > 0) std::memcpy(v, t_bell.h + 16, nv * sizeof(double));
  return SP_OK;
}

// `need` < 0: the caller needs every kept triplet (the SVD projector);
// need >= 0: only the leading `need` triplets and whether the kept rank
// reaches them (the ID lifting).  For the latter, a block whose spectrum is
// still above the cut at its last column does not grow once it holds need + 8
// values, and values within 10x of the block's tail (an unresolved bulk, e.g.
// the noise floor of cfg3) are exempt from the stability test.
// Ypre (rows x 32, ld 32, may be null): the SRHT test block of width 32
// already formed (fused with the gather of X, srht_gather); used for the
// first block when it has that width.
static int svd_top(const double* X, int64_t rows, int64_t cols, int64_t ldx, int want, double power,
                   TopSvd& out, Arena& ar, cudaStream_t s, PendingFlag pf = PendingFlag(), bool want_v = false,
                   int need = -1, const double* Ypre = nullptr) {
  const int64_t p = std::min(rows, cols);
  int hflag = 0;
  if (p <= 64 && pf.dev) {
    // the exact path checks finiteness itself (thin_svd); surface the caller's message
    if (pf.check_input) SPB_TRY(check_finite_async(rows, cols, X, ldx, pf.dev, s));
    PinnedReads rd(s);
    SPB_TRY(read_flag_with(pf, hflag, rd));
    SPB_TRY(rd.sync());
    if (hflag) {
      set_error(pf.msg);
      return SP_ENUMERICAL;
    }
  }
  // the exact SVD of X (size-general thin_svd: TSQR / blocked QR + Jacobi)
  auto exact = [&]() -> int {
    out.b = (int)p;
    out.iters = 0;
    out.U = ar.alloc<double>((size_t)rows * p);
    out.S = ar.alloc<double>((size_t)p);
    out.V = ar.alloc<double>((size_t)cols * p);
    if (ar.failed()) {
      set_error("svd_top workspace allocation failed");
      return SP_ECUDA;
    }
    SPB_TRY(thin_svd(rows, cols, X, ldx, out.U, p, out.S, out.V, p, s));
    out.hs.resize(p);
    SPB_TRY(read_small(out.hs.data(), out.S, p * sizeof(double), s));
    out.kept = count_kept(out.hs, power);
    return SP_OK;
  };
  if (p <= 64) return exact();
  auto exact_fallback = [&]() -> int {
    if (pf.dev && pf.check_input) {  // the randomized path's input check already ran
      PinnedReads rd(s);
      SPB_TRY(read_flag_with(pf, hflag, rd));
      SPB_TRY(rd.sync());
      if (hflag) {
        set_error(pf.msg);
        return SP_ENUMERICAL;
      }
    }
    return exact();
  };
  const int cap = (int)std::min<int64_t>(p, 256);
  int b = std::min(cap, (std::max(32, want + 16) + 7) / 8 * 8);
  for (;;) {
    Arena it(s);
    double* Om = it.alloc<double>((size_t)cols * b);
    double* Y = it.alloc<double>((size_t)rows * b);
    double* Q = it.alloc<double>((size_t)rows * b);
    double* Z = it.alloc<double>((size_t)cols * b);
    double* P = it.alloc<double>((size_t)cols * b);
    double* Rt = it.alloc<double>((size_t)b * b);
    double* Rz = it.alloc<double>((size_t)b * b);
    double* Us = it.alloc<double>((size_t)b * b);
    double* Vs = it.alloc<double>((size_t)b * b);
    double* Sg = it.alloc<double>((size_t)b);
    if (it.failed()) {
      set_error("svd_top workspace allocation failed");
      return SP_ECUDA;
    }
    // test block: subsampled randomized Hadamard transform of the rows of X
    // (srht.cu, also the finite check of X) when the width allows, else a
    // dense uniform block on the DMMA GEMM (finite check on Y)
    int* xflag = (pf.dev && pf.check_input) ? pf.dev : nullptr;
    const double* Y0 = Y;  // the first test block
    if (Ypre && b == 32) {
      Y0 = Ypre;
    } else if (srht_sketch(rows, cols, X, ldx, b, kSrhtSeed + (uint64_t)b, Y, b, xflag, s) != SP_OK) {
      SPB_TRY(fill_uniform(cols, b, Om, b, 0x5eed5eedull + (uint64_t)b, s));
      SPB_TRY(gemm(0, 0, rows, b, cols, 1.0, X, ldx, Om, b, 0.0, Y, b, s));
      if (xflag) SPB_TRY(check_finite_async(rows, b, Y, b, xflag, s));
    }
    SPB_TRY(tsqr(rows, b, Y0, b, Q, b, Rt, b, s));
    std::vector<double> prev, hs(b);
    int kept_prev = -1, kept = 0, iters = 0;
    bool grow = false;
    const int max_it = 24;
    // outputs for this block width (the speculative final products below)
    double* oU = ar.alloc<double>((size_t)rows * b);
    double* oS = ar.alloc<double>((size_t)b);
    double* oV = want_v ? ar.alloc<double>((size_t)cols * b) : nullptr;
    if (ar.failed()) {
      set_error("svd_top workspace allocation failed");
      return SP_ECUDA;
    }
    auto final_products = [&](bool copy_s) -> int {
      SPB_TRY(gemm(0, 0, rows, b, b, 1.0, Q, b, Us, b, 0.0, oU, b, s));
      if (want_v) SPB_TRY(gemm(0, 0, cols, b, b, 1.0, P, b, Vs, b, 0.0, oV, b, s));
      if (copy_s) SPB_CUDA(cudaMemcpyAsync(oS, Sg, b * sizeof(double), cudaMemcpyDeviceToDevice, s));
      return SP_OK;
    };
    bool spec = false, conv_seen = false;
    int bulk_from = 0;
    for (int itn = 0; itn < max_it; ++itn) {
      // Rayleigh-Ritz: Q^T X = Z^T with Z = X^T Q = P Rz  ->  Q^T X = Rz^T P^T
      // Z = P Rz: only Rz is needed unless V is wanted (R alone: Cholesky of
      // the double-double Gram, ddgram.cu -- one launch instead of the 32-step
      // Householder factor; it sums the split-K slabs of Z itself, and Z is
      // reduced explicitly only if another step follows)
      const bool lazy_p = b <= 32 && !want_v && gram_chol_dd_ok(cols, b);
      double* Zp = nullptr;
      int zs = 0;
      if (lazy_p) {
        SPB_TRY(gemm_partials(1, 0, cols, b, rows, X, ldx, Q, b, it, &Zp, &zs, s));
        SPB_TRY(gram_chol_dd(cols, b, Zp, b, Rz, b, it, s, zs, (int64_t)cols * b));
      } else {
        SPB_TRY(gemm(1, 0, cols, b, rows, 1.0, X, ldx, Q, b, 0.0, Z, b, s));
        SPB_TRY(tsqr(cols, b, Z, b, P, b, Rz, b, s));
      }
      SPB_TRY(jacobi_svd_tr(b, Rz, b, /*trans=*/true, Us, b, Sg, want_v ? Vs : nullptr, b, s));
      // publish the Ritz values, then -- while the host waits for them --
      // form the final products as if this step converged (it usually does;
      // otherwise they are recomputed after the next step)
      // (only when they are cheap: a wasted product must not cost more than
      // the host round trip it hides)
      spec = (double)b * b * (rows + (want_v ? cols : 0)) <= 64.0 * 1024 * 1024;
      unsigned seq = 0;
      host_mark("svd_top: rr launched");
      SPB_TRY(bell_publish(Sg, b, itn == 0 ? pf.dev : nullptr, seq, s, oS));
      if (spec) SPB_TRY(final_products(false));
      host_mark("svd_top: spin");
      SPB_TRY(bell_wait(seq, hs.data(), b, &hflag, s));
      host_mark("svd_top: spectrum in");
      if (!(itn == 0 && pf.dev)) hflag = 0;
      if (hflag) {
        set_error(pf.msg);
        return SP_ENUMERICAL;
      }
      iters = itn + 1;
      kept = count_kept(hs, power);
      if (kept + 8 > b && (need < 0 || kept < need + 8)) {
        if (b < cap) {
          grow = true;
          break;
        }
        // the block cannot hold every kept direction plus oversampling: never
        // return a truncated projector (the reference keeps its full QR basis)
        return exact_fallback();
      }
      bool conv = false;
      if (need >= 0) {
        // ID mode: the leading t = min(kept, need) triplets feed the lifting
        // V_t S_t^-1 U_t^T A and must be converged as a subspace.  Subspace
        // iteration resolves them at the rate rho = sigma_{b-7} / sigma_t per
        // step (angle ~rho^(2 itn + 2) after itn + 1 Rayleigh-Ritz steps):
        // stop at 1e-12; when more than 8 further steps would be needed, grow
        // the block (rho falls with b); a flat stretch of the spectrum at t
        // that even the largest block cannot resolve (a noise bulk: cfg3's
        // r = 200 split, cfg5's FP32 floor) takes the exact SVD of X up to
        // kExactMax columns, else is accepted and flagged (bulk).
        const int t = std::min(kept, need);
        if (t == 0) {
          conv = true;
        } else {
          const double rho = hs[b - 8] / hs[t - 1];
          if ((itn == 0 && rho <= 1e-8) || (itn >= 1 && kept_prev >= t && std::pow(rho, 2.0 * itn + 2.0) <= 1e-12)) {
            conv = true;
          } else {
            const double more = rho < 1.0 ? (std::log(1e-12) / std::log(rho) - 2.0) / 2.0 - itn : 1e9;
            if (more > 8.0) {
              // a flat stretch (rho > 0.95: a noise bulk) does not become
              // resolvable with a wider block -- only a slowly decaying one does
              if (b < cap && rho <= 0.95) {
                grow = true;
                break;
              }
              if (p <= kExactMax && std::max(rows, cols) <= kExactLong) return exact_fallback();
              if (!out.bulk) bulk_from = itn;
              out.bulk = true;  // a few more steps: the Ritz values above the stretch settle
            }
          }
          if (!conv && out.bulk && itn >= 1) {
            conv = itn - bulk_from >= 3;
            if (!conv) {
              conv = true;
              for (int i = 0; i < std::min(b, need); ++i) {
                if (hs[i] <= 10.0 * hs[b - 1]) break;  // the flat stretch itself
                if (std::fabs(hs[i] - prev[i]) > 1e-12 * hs[i]) conv = false;
              }
            }
          }
        }
        if (conv) {
          conv_seen = true;
          break;
        }
        prev = hs;
        kept_prev = kept;
      }
      // One Rayleigh-Ritz step already resolves the kept triplets to
      // (sigma_{b+1}/sigma_kept)^2 when the spectrum has fallen to the
      // rounding floor inside the block (oversampling 8): accept it.
      if (need < 0) {
        if (itn == 0 && kept > 0 && b - 8 > kept && hs[b - 8] <= 1e-8 * hs[kept - 1]) conv = true;
        // A priori: after itn + 1 Rayleigh-Ritz steps the kept subspace is within
        // an angle ~rho^(2 itn) of the exact one, rho = sigma_{b-7} / sigma_kept
        // (oversampling 8; hs[b-8] >= sigma_{b+1} makes the estimate
        // conservative), and the kept Ritz values within its square.  Stop once
        // rho^(2 itn + 2) <= 1e-12: an angle below ~1e-11, whose effect on the
        // singular values of P_r A is second order (~1e-22 sigma_1) and far
        // inside the 1e-8 principal-angle gate (measured on the cfg3 sketch,
        // whose noise bulk gives rho = 0.18: 7e-12 when the test first passes;
        // the earlier 1e-16 bound ran three more steps for nothing).  An
        // FP32-stored A floors the sketch spectrum at ~1e-7 sigma_1: rho ~1e-4
        // and the second step passes.
        if (itn >= 1 && kept == kept_prev && kept > 0 && b - 8 > kept &&
            std::pow(hs[b - 8] / hs[kept - 1], 2.0 * itn + 2.0) <= 1e-12)
          conv = true;
        if (!conv && itn >= 1 && kept == kept_prev) {
          conv = true;
          const int chk = std::min(b, kept + 1);
          for (int i = 0; i < chk; ++i)
            if (std::fabs(hs[i] - prev[i]) > 1e-14 * hs[0] + 1e-12 * hs[i]) conv = false;
        }
        if (conv) {
          conv_seen = true;
          break;
        }
        prev = hs;
        kept_prev = kept;
      }
      // one more subspace iteration, started from the Ritz vectors:
      // Y = X (Z Us) = X P Vs Sigma (Z = P Rz, Rz^T = Us Sigma Vs^T; the column
      // scaling leaves the span and the column-wise backward-stable Householder
      // QR unchanged), Q = orth(Y).  Q then arrives nearly aligned with the
      // singular vectors, so the next core Rz is nearly diagonal and its Jacobi
      // SVD takes a few sweeps instead of ~8 (a noise bulk in the block is
      // nearly invariant under X X^T, so it stays nearly diagonal too).  P is
      // scratch here: the next step recomputes it.
      if (lazy_p) {  // Z itself is needed now
        if (zs > 1)
          SPB_TRY(split_reduce(Zp, zs, cols, b, 1.0, 0.0, Z, b, s));
        else
          SPB_TRY(copy2d(cols, b, Zp, b, Z, b, s));
      }
      static const bool plain_restart = getenv("SPB_RR_PLAIN") != nullptr;  // experiments: Y = X P
      if (plain_restart) {
        if (lazy_p) {
          TsqrPlan zplan;
          SPB_TRY(tsqr_factor(cols, b, Z, b, Rz, b, zplan, it, s));
          SPB_TRY(tsqr_form_q(zplan, P, b, it, s));
        }
      } else {
        SPB_TRY(gemm(0, 0, cols, b, b, 1.0, Z, b, Us, b, 0.0, P, b, s));
      }
      SPB_TRY(gemm(0, 0, rows, b, cols, 1.0, X, ldx, P, b, 0.0, Y, b, s));
      SPB_TRY(tsqr(rows, b, Y, b, Q, b, Rt, b, s));
      // Blind steps.  The first Rayleigh-Ritz step gives the contraction rate
      // rho = sigma_{b-7} / sigma_kept, hence the step at which the a-priori
      // test above can first pass.  The steps in between need no Ritz values
      // and no host decision: plain simultaneous iteration Q <- orth(X X^T Q)
      // from the Ritz-aligned start (Householder QR keeps the nested column
      // spans, so the columns stay aligned with the singular directions and
      // the small kept ones keep their column-relative accuracy); the last two
      // steps are Rayleigh-Ritz steps again (kept == kept_prev, Ritz values,
      // the rate test with the then-current spectrum -- an optimistic rho only
      // costs further Rayleigh-Ritz steps).  Per blind step: two products and
      // a TSQR instead of those plus the dd Gram, the Jacobi core, the
      // doorbell round trip and the restart product (cfg3: 250 vs 414 us).
      static const bool no_blind = getenv("SPB_RR_EVERY_STEP") != nullptr;
      // ID mode: the same between the first step and the step at which the
      // leading-triplet rate test can first pass; in bulk mode (accepted
      // itn - bulk_from >= 3 steps after the flat stretch was found) the two
      // steps in between.
      // After ANY unconverged Rayleigh-Ritz step (its rho is the current, better
      // estimate): blind steps up to two before the predicted passing step, at
      // most kBlindMax in a row -- a slowly contracting block still sees a
      // Rayleigh-Ritz step (stagnation test, block growth) every kBlindMax + 1.
      constexpr int kBlindMax = 6;
      int blind = 0;
      if (!no_blind && need < 0 && kept > 0 && b - 8 > kept) {
        const double rho = hs[b - 8] / hs[kept - 1];
        if (rho > 0.0 && rho < 1.0)
          blind = (int)std::ceil((std::log(1e-12) / std::log(rho) - 2.0) / 2.0) - 2 - itn;
      } else if (!no_blind && need >= 0 && out.bulk && itn == bulk_from) {
        blind = 2;
      } else if (!no_blind && need >= 0 && !out.bulk && std::min(kept, need) > 0) {
        const double rho = hs[b - 8] / hs[std::min(kept, need) - 1];
        if (rho > 0.0 && rho < 1.0)
          blind = std::max(1, (int)std::ceil((std::log(1e-12) / std::log(rho) - 2.0) / 2.0)) - 2 - itn;
      }
      blind = std::min(blind, kBlindMax);
      blind = std::min(blind, max_it - 3 - itn);
      for (int j = 0; j < blind; ++j) {
        SPB_TRY(gemm(1, 0, cols, b, rows, 1.0, X, ldx, Q, b, 0.0, Z, b, s));
        SPB_TRY(gemm(0, 0, rows, b, cols, 1.0, X, ldx, Z, b, 0.0, Y, b, s));
        SPB_TRY(tsqr(rows, b, Y, b, Q, b, Rt, b, s));
        ++itn;
      }
    }
    if (grow) {
      b = std::min(cap, 2 * b);
      continue;
    }
    if (!conv_seen && !out.bulk) return exact_fallback();  // max_it exhausted without convergence
    if (!spec) SPB_TRY(final_products(false));  // oS was written by the publication
    out.b = b;
    out.kept = kept;
    out.iters = iters;
    out.hs = hs;
    out.U = oU;
    out.S = oS;
    out.V = oV;
    return SP_OK;
  }
}

// Per-thread side stream (+ fork / join events) for independent small chains.
struct AuxStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  int dev = -1;
};

static AuxStream& aux_stream() {
  static thread_local AuxStream ax[16];
  int dev = 0;
  cudaGetDevice(&dev);
  AuxStream& a = ax[dev & 15];
  if (a.s == nullptr || a.dev != dev) {
    cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming);
    a.dev = dev;
  }
  return a;
}

// ----------------------------------------------------- deferred status ----
// The fused finish stage never synchronises; its device flag (Cholesky
// breakdown / non-finite input) is copied to pinned memory behind the call's
// last kernel and read by sp_deferred_status() after the caller's own sync
// (the host-result API does this right after its device->host copies and
// re-runs the call with the Householder finish when it is set).
struct Deferred {
  int* host = nullptr;
  cudaEvent_t ev = nullptr;
  bool pending = false;
};
static thread_local Deferred t_def;
static thread_local int t_finish_mode = 0;  // 1: Householder TSQR finish

// Per-stream {flag, ticket} words of the fused finish: zeroed once at
// creation; the ticket is reset by the Gram tail that consumes it and the flag
// behind its deferred read (at the end of the call), so no memset node sits
// inside the call's chain of dependent launches.
static int finish_words(cudaStream_t s, int** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, int*> words;
  int dev = 0;
  SPB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = words.find({dev, s});
  if (it == words.end()) {
    int* p = nullptr;
    SPB_CUDA(cudaMalloc(&p, 2 * sizeof(int)));
    SPB_CUDA(cudaMemsetAsync(p, 0, 2 * sizeof(int), s));
    it = words.emplace(std::make_pair(dev, s), p).first;
  }
  *out = it->second;
  return SP_OK;
}

// The fused finish publishes its status word itself (finish_core writes the
// mapped pinned word and rezeroes the device flag): get the device view of
// the host word before the launches, record the completion event after them.
static int defer_begin(int** hdev) {
  if (!t_def.host) {
    SPB_CUDA(cudaHostAlloc(&t_def.host, sizeof(int), cudaHostAllocMapped));
    SPB_CUDA(cudaEventCreateWithFlags(&t_def.ev, cudaEventDisableTiming));
  }
  if (t_def.pending) SPB_CUDA(cudaEventSynchronize(t_def.ev));  // previous value is superseded
  SPB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(hdev), t_def.host, 0));
  return SP_OK;
}
static int defer_end(cudaStream_t s) {
  SPB_CUDA(cudaEventRecord(t_def.ev, s));
  t_def.pending = true;
  return SP_OK;
}

int deferred_status(int* out) {
  *out = 0;
  if (!t_def.pending) return SP_OK;
  SPB_CUDA(cudaEventSynchronize(t_def.ev));
  *out = *t_def.host;
  t_def.pending = false;
  return SP_OK;
}

void set_finish_mode(int mode) { t_finish_mode = mode; }

bool finish_fused_ok(int64_t m, int64_t n, int r, int k);
int finish_fused(int64_t m, int64_t n, const double* Z, int64_t ldz, const double* Y, int r, int k, double* U,
                 double* S, double* V, int* dflag, int* hflag, cudaStream_t s);

// Given the kept left basis Z (m x r, ld ldz) of the sketch, one read of A:
// Y = A^T Z, then the rank-k SVD of Z Z^T A written to U (m x k), S, V (n x k).
static int finish_svd(const void* A, int a_dtype, int64_t m, int64_t n, int64_t lda, const double* Z,
                      int64_t ldz, int r, int k, double* U, double* S, double* V, double kappa_est,
                      cudaStream_t s, bool* fused) {
  Arena ar(s);
  *fused = false;
  if (r > 0 && t_finish_mode == 0 && kappa_est < 1e6 && finish_fused_ok(m, n, r, k)) {
    *fused = true;
    // A pass + fused shifted-CholeskyQR2 / Jacobi / completion: no host sync
    SPB_ALLOC(ar, double, Y, (size_t)n * r);
    int* dflag = nullptr;  // {flag, ticket}, zero on entry
    SPB_TRY(finish_words(s, &dflag));
    int* hflag = nullptr;
    SPB_TRY(defer_begin(&hflag));
    host_mark("finish: A pass launch");
    SPB_TRY(skinny_atz(A, a_dtype, m, n, lda, Z, ldz, r, Y, r, s));
    host_mark("finish: A pass launched");
    SPB_TRY(finish_fused(m, n, Z, ldz, Y, r, k, U, S, V, dflag, hflag, s));
    host_mark("finish: launched");
    SPB_TRY(defer_end(s));  // finish_core published the flag and rezeroed dflag[0]
    return SP_OK;
  }
  SPB_CUDA(cudaMemsetAsync(S, 0, k * sizeof(double), s));
  const int kk = std::min(r, k);
  if (r > 0) {
    SPB_ALLOC(ar, double, Y, (size_t)n * r);
    SPB_ALLOC(ar, double, Qy, (size_t)n * r);
    SPB_ALLOC(ar, double, Ry, (size_t)r * r);
    SPB_ALLOC(ar, double, Us, (size_t)r * r);
    SPB_ALLOC(ar, double, Vs, (size_t)r * r);
    SPB_ALLOC(ar, double, Sr, (size_t)r);
    SPB_TRY(skinny_atz(A, a_dtype, m, n, lda, Z, ldz, r, Y, r, s));     // the A pass
    // A non-finite entry of A outside the sketch columns passes every
    // sketch-side check and first shows up here, in Y = A^T Z; the reference
    // raises it from thin_svd(projected) (src/kernels.py:87-91).  Raised as a
    // device flag read together with the CholeskyQR2 breakdown flag (one read).
    SPB_ALLOC(ar, int, yflag, 2);
    SPB_CUDA(cudaMemsetAsync(yflag, 0, 2 * sizeof(int), s));
    SPB_TRY(check_finite_async(n, r, Y, r, yflag, s));
    // kappa(Y) ~ the kept spectral range: CholeskyQR2 below 1e6 (breakdown is
    // checked once at the end, and the factorisation redone by Householder
    // TSQR if it happened), else Householder TSQR directly
    const bool chol = kappa_est < 1e6 && r <= 112 && t_finish_mode == 0;
    int* qflag = nullptr;
    if (chol) {
      qflag = yflag + 1;
      SPB_TRY(cholqr2_async(n, r, Y, r, Qy, r, Ry, r, qflag, s));
    } else {
      SPB_TRY(tsqr(n, r, Y, r, Qy, r, Ry, r, s));
    }
    bool y_checked = false;
  retry:
    SPB_TRY(jacobi_svd_tr(r, Ry, r, /*trans=*/true, Us, r, Sr, Vs, r, s));  // Ry^T = Us Sr Vs^T
    if (!y_checked) {
      int h[2] = {0, 0};
      SPB_TRY(read_small(h, yflag, 2 * sizeof(int), s));
      y_checked = true;
      if (h[0]) {
        set_error("SVD input contains non-finite entries");
        return SP_ENUMERICAL;
      }
      if (qflag && h[1]) {  // CholeskyQR2 broke down: Householder TSQR and redo the core
        qflag = nullptr;
        SPB_TRY(tsqr(n, r, Y, r, Qy, r, Ry, r, s));
        goto retry;
      }
    }
    if (r < k && product_with_completion_ok(m, r, k) && product_with_completion_ok(n, r, k)) {
      // U = [Z Us | completion], V = [Qy Vs | completion], one pass each; the
      // (short, latency-bound) U chain runs on a side stream beside V's
      AuxStream& ax = aux_stream();
      SPB_CUDA(cudaEventRecord(ax.fork, s));
      SPB_CUDA(cudaStreamWaitEvent(ax.s, ax.fork, 0));
      SPB_TRY(product_with_completion(m, r, k, Z, ldz, Us, r, U, k, ax.s));
      SPB_TRY(product_with_completion(n, r, k, Qy, r, Vs, r, V, k, s));
      SPB_CUDA(cudaEventRecord(ax.join, ax.s));
      SPB_CUDA(cudaStreamWaitEvent(s, ax.join, 0));
      SPB_CUDA(cudaMemcpyAsync(S, Sr, kk * sizeof(double), cudaMemcpyDeviceToDevice, s));
      return SP_OK;
    }
    if (r <= k) {
      SPB_TRY(gemm(0, 0, m, r, r, 1.0, Z, ldz, Us, r, 0.0, U, k, s));     // U = Z Us
      SPB_TRY(gemm(0, 0, n, r, r, 1.0, Qy, r, Vs, r, 0.0, V, k, s));      // V = Qy Vs
    } else {
      SPB_ALLOC(ar, double, Uf, (size_t)m * r);
      SPB_ALLOC(ar, double, Vf, (size_t)n * r);
      SPB_TRY(gemm(0, 0, m, r, r, 1.0, Z, ldz, Us, r, 0.0, Uf, r, s));
      SPB_TRY(gemm(0, 0, n, r, r, 1.0, Qy, r, Vs, r, 0.0, Vf, r, s));
      SPB_TRY(copy2d(m, kk, Uf, r, U, k, s));
      SPB_TRY(copy2d(n, kk, Vf, r, V, k, s));
    }
    SPB_CUDA(cudaMemcpyAsync(S, Sr, kk * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  SPB_TRY(complete_basis(m, kk, k, U, k, 0xC0FFEEull, s));
  SPB_TRY(complete_basis(n, kk, k, V, k, 0xBEEFull, s));
  return SP_OK;
}

// ----------------------------------------------------------- sketching ----
__global__ void same_set_kernel(const int64_t* idx, const double* w, const int64_t* cols, int64_t n,
                                int* differ) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (idx[i] != cols[i] || w[i] != 1.0) atomicOr(differ, 1);
}

// Is the sketch s0 = A D bit-identical to C = A(:, cols)?  (depth-1 unit
// weights, no projection, idx == cols.)  Synchronises.
static int sketch_is_columns(const int64_t* idx, const double* w, int depth, int64_t nc,
                             const double* omega, const int64_t* cols, int64_t ncols, bool& same,
                             cudaStream_t s) {
  same = false;
  if (depth != 1 || omega != nullptr || nc != ncols || cols == nullptr) return SP_OK;
  Arena ar(s);
  SPB_ALLOC(ar, int, differ, 1);
  SPB_CUDA(cudaMemsetAsync(differ, 0, sizeof(int), s));
  same_set_kernel<<<ceil_div(nc, 256), 256, 0, s>>>(idx, w, cols, nc, differ);
  count_launch();
  SPB_CHECK_LAUNCH();
  int h = 1;
  SPB_TRY(read_small(&h, differ, sizeof(int), s));
  same = (h == 0);
  return SP_OK;
}

// s0 = (A D) [omega]  (m x out_dim)
static int make_sketch(const void* A, int a_dtype, int64_t m, int64_t n, int64_t lda, const int64_t* idx,
                       const double* w, int depth, int64_t nc, const double* omega, int64_t ell,
                       double* s0, Arena& ar, cudaStream_t s) {
  if (!omega) return apply_stencil(A, a_dtype, m, n, lda, idx, w, depth, nc, false, s0, nc, s);
  double* tmp = ar.alloc<double>((size_t)m * nc);
  if (!tmp) {
    set_error("sketch workspace allocation failed");
    return SP_ECUDA;
  }
  SPB_TRY(apply_stencil(A, a_dtype, m, n, lda, idx, w, depth, nc, false, tmp, nc, s));
  return gemm(0, 0, m, ell, nc, 1.0, tmp, nc, omega, ell, 0.0, s0, ell, s);
}

static void fill_info(int64_t* info, int kept, int warn, const TopSvd& t, int64_t launches0) {
  if (!info) return;
  for (int i = 0; i < SP_INFO_LEN; ++i) info[i] = 0;
  info[SP_INFO_KEPT] = kept;
  info[SP_INFO_WARN] = warn;
  info[SP_INFO_BLOCK] = t.b;
  info[SP_INFO_ITERS] = t.iters;
  info[SP_INFO_LAUNCHES] = launches() - launches0;
}

// --------------------------------------------------------- single_pass_svd ----
int single_pass_svd(const void* A, int a_dtype, int64_t m, int64_t n, int64_t lda, const int64_t* idx,
                    const double* w, int depth, int64_t nc, const double* omega, int64_t ell, int k,
                    const double* pre_s0, double* U, double* S, double* V, int64_t* info,
                    cudaStream_t s) {
  const int64_t l0 = launches();
  const int64_t out_dim = omega ? ell : nc;
  // src/svd.py:71-77
  SPB_REQUIRE(k >= 1, "target rank k must be >= 1");
  SPB_REQUIRE(k <= out_dim, "target rank k=" + std::to_string(k) + " exceeds sketch width n_c=" + std::to_string(out_dim));
  SPB_REQUIRE(k <= std::min(m, out_dim), "target rank k=" + std::to_string(k) + " exceeds min(m, n_c)");
  Arena ar(s);
  const double* s0 = pre_s0;
  if (!s0) {
    double* t = ar.alloc<double>((size_t)m * out_dim);
    if (!t) {
      set_error("sketch allocation failed");
      return SP_ECUDA;
    }
    SPB_TRY(make_sketch(A, a_dtype, m, n, lda, idx, w, depth, nc, omega, ell, t, ar, s));
    s0 = t;
  }
  SPB_ALLOC(ar, int, fflag, 1);
  SPB_CUDA(cudaMemsetAsync(fflag, 0, sizeof(int), s));
  TopSvd top;
  PendingFlag pf;
  pf.dev = fflag;
  pf.check_input = true;
  pf.msg = "QR input contains non-finite entries";
  SPB_TRY(svd_top(s0, m, out_dim, out_dim, 1, 1.0, top, ar, s, pf));
  const int r = top.kept;
  const double kappa = (r > 0 && top.hs[r - 1] > 0.0) ? top.hs[0] / top.hs[r - 1] : INFINITY;
  bool fused = false;
  SPB_TRY(finish_svd(A, a_dtype, m, n, lda, top.U, top.b, r, k, U, S, V, kappa, s, &fused));
  const bool healthy = (m >= out_dim) && (r == out_dim);
  fill_info(info, r, healthy ? 0 : SP_WARN_RANK_DEFICIENT, top, l0);
  if (info) info[SP_INFO_FUSED] = fused ? 1 : 0;
  return SP_OK;
}

// ------------------------------------------------------------- power_svd ----
int power_svd(const void* A, int a_dtype, int64_t m, int64_t n, int64_t lda, const int64_t* idx,
              const double* w, int depth, int64_t nc, const double* omega, int64_t ell,
              const int64_t* cols, int64_t ncols, int q, int k, const double* pre_s0,
              const double* pre_c, int hints, double* U, double* S, double* V, int64_t* info,
              cudaStream_t s) {
  host_mark("power_svd enter");
  const int64_t l0 = launches();
  const int64_t out_dim = omega ? ell : nc;
  // src/power.py:235-241, 216-224, 330-331
  SPB_REQUIRE(k <= out_dim, "target rank k=" + std::to_string(k) + " exceeds sketch width " + std::to_string(out_dim));
  SPB_REQUIRE(cols != nullptr && ncols > 0, "column index set out of range");
  SPB_REQUIRE(ncols > k, "column set size " + std::to_string(ncols) + " must exceed target rank " + std::to_string(k));
  SPB_REQUIRE(ncols >= out_dim, "column set size " + std::to_string(ncols) + " must cover the sketch width " + std::to_string(out_dim));
  SPB_REQUIRE(q >= 1, "single-pass power pipeline needs q >= 1");
  if (!(hints & SP_HINT_COLS_VALIDATED)) SPB_TRY(check_columns(cols, ncols, n, s));
  SPB_REQUIRE(k >= 1 && k <= std::min(m, out_dim),
              "target rank k=" + std::to_string(k) + " outside the enriched basis width");
  Arena ar(s);
  bool same = false;
  if (hints & SP_HINT_SAME_SET)
    same = true;
  else if (!(hints & SP_HINT_DIFFERENT_SET))
    SPB_TRY(sketch_is_columns(idx, w, depth, nc, omega, cols, ncols, same, s));
  SPB_ALLOC(ar, int, fflag, 1);
  SPB_CUDA(cudaMemsetAsync(fflag, 0, sizeof(int), s));
  const double* C = pre_c;
  const double* Ypre = nullptr;
  if (!C) {
    double* t = ar.alloc<double>((size_t)m * ncols);
    if (!t) {
      set_error("column block allocation failed");
      return SP_ECUDA;
    }
    if (same && std::min<int64_t>(m, ncols) > 64 && srht_gather_ok(m, ncols, 32)) {
      // K1 fused with the range finder's test block: C and Y = C D H S in one pass
      double* y = ar.alloc<double>((size_t)m * 32);
      if (!y) {
        set_error("test block allocation failed");
        return SP_ECUDA;
      }
      host_mark("gather launch");
      SPB_TRY(srht_gather(A, a_dtype, m, lda, cols, ncols, t, ncols, 32, kSrhtSeed + 32, y, 32, fflag, s));
      host_mark("gather launched");
      Ypre = y;
    } else {
      SPB_TRY(apply_stencil(A, a_dtype, m, n, lda, cols, nullptr, 1, ncols, true, t, ncols, s));
    }
    C = t;
  }
  TopSvd top;
  if (same) {
    PendingFlag pf;
    pf.dev = fflag;
    pf.check_input = true;
    pf.msg = "power iterate overflowed; enable re-orthonormalization (reorth)";
    SPB_TRY(svd_top(C, m, ncols, ncols, 1, 2.0 * q + 1.0, top, ar, s, pf, false, -1, Ypre));
    // the reference forms G = (C C^T)^q C explicitly and raises once it
    // overflows (src/power.py:81-85); G is never formed here, so mirror the
    // condition on its largest singular value sigma_1(C)^(2q+1)
    if (!top.hs.empty() && !std::isfinite(std::pow(top.hs[0], 2.0 * q + 1.0))) {
      set_error("power iterate overflowed; enable re-orthonormalization (reorth)");
      return SP_ENUMERICAL;
    }
  } else {
    const double* s0 = pre_s0;
    if (!s0) {
      double* t = ar.alloc<double>((size_t)m * out_dim);
      if (!t) {
        set_error("sketch allocation failed");
        return SP_ECUDA;
      }
      SPB_TRY(make_sketch(A, a_dtype, m, n, lda, idx, w, depth, nc, omega, ell, t, ar, s));
      s0 = t;
    }
    // G = (C C^T)^q s0 in the reference's association (src/power.py:99-108)
    double* G = ar.alloc<double>((size_t)m * out_dim);
    double* T = ar.alloc<double>((size_t)ncols * out_dim);
    if (ar.failed()) {
      set_error("power iterate allocation failed");
      return SP_ECUDA;
    }
    SPB_TRY(copy2d(m, out_dim, s0, out_dim, G, out_dim, s));
    for (int it = 0; it < q; ++it) {
      SPB_TRY(gemm(1, 0, ncols, out_dim, m, 1.0, C, ncols, G, out_dim, 0.0, T, out_dim, s));
      SPB_TRY(check_finite(ncols, out_dim, T, out_dim, "power iterate overflowed; enable re-orthonormalization (reorth)", s));
      SPB_TRY(gemm(0, 0, m, out_dim, ncols, 1.0, C, ncols, T, out_dim, 0.0, G, out_dim, s));
      SPB_TRY(check_finite(m, out_dim, G, out_dim, "power iterate overflowed; enable re-orthonormalization (reorth)", s));
    }
    SPB_TRY(svd_top(G, m, out_dim, out_dim, 1, 1.0, top, ar, s));
  }
  const int r = top.kept;
  const double kappa = (r > 0 && top.hs[r - 1] > 0.0) ? top.hs[0] / top.hs[r - 1] : INFINITY;
  bool fused = false;
  SPB_TRY(finish_svd(A, a_dtype, m, n, lda, top.U, top.b, r, k, U, S, V, kappa, s, &fused));
  const bool healthy = (m >= out_dim) && (r == out_dim);
  fill_info(info, r, healthy ? 0 : SP_WARN_RANK_DEFICIENT, top, l0);
  if (info) info[SP_INFO_FUSED] = fused ? 1 : 0;
  return SP_OK;
}

// ------------------------------------------------------- sketch basis ----
// Kept left basis of a sketch-sized X (the svd_top + kept-rank step of the
// pipelines, exported for the column-sharded driver): U (rows x min(r, r_max)),
// S; info[KEPT] = r = #{(s_i/s_1)^power > 1e-12}.
int sketch_basis(const double* X, int64_t rows, int64_t cols, int64_t ldx, double power, int r_max, double* U,
                 int64_t ldu, double* S, int64_t* info, cudaStream_t s) {
  const int64_t l0 = launches();
  SPB_REQUIRE(rows >= 1 && cols >= 1 && r_max >= 1, "sketch_basis needs a non-empty matrix");
  Arena ar(s);
  SPB_ALLOC(ar, int, fflag, 1);
  SPB_CUDA(cudaMemsetAsync(fflag, 0, sizeof(int), s));
  PendingFlag pf;
  pf.dev = fflag;
  pf.check_input = true;
  pf.msg = "sketch contains non-finite entries";
  TopSvd top;
  SPB_TRY(svd_top(X, rows, cols, ldx, 1, power, top, ar, s, pf));
  const int r = std::min(top.kept, r_max);
  if (r > 0) {
    SPB_TRY(copy2d(rows, r, top.U, top.b, U, ldu, s));
    SPB_CUDA(cudaMemcpyAsync(S, top.S, r * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  fill_info(info, top.kept, 0, top, l0);
  return SP_OK;
}

// ---------------------------------------------------------------- row ID ----
__global__ void scatter_p_kernel(int64_t m, int k, const int64_t* perm, const double* coef, int64_t ldc,
                                 double* P) {
  // P[perm[i], :] = e_i (i < k); P[perm[k + j], :] = coef[:, j]^T
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * k) return;
  const int64_t row = e / k;
  const int c = (int)(e % k);
  const int64_t dst = perm[row];
  P[dst * k + c] = (row < k) ? (row == c ? 1.0 : 0.0) : coef[(int64_t)c * ldc + (row - k)];
}

__global__ void gather_rows_kernel(const int64_t* rows_idx, int k, const double* X, int64_t ldx, int64_t cols,
                                   double* out, int64_t ldo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)k * cols) return;
  const int64_t i = e / cols, c = e % cols;
  out[i * ldo + c] = X[rows_idx[i] * ldx + c];
}

// Interpolation coefficients from a rank-k pivoted QR of M^T (perm: pivot
// order over the m candidates, R: k x m with R[:, perm-order]):
// C = R1^-1 R2, or the pseudo-inverse solve when R1 is rank deficient
// (src/rowid.py:60-75); P[perm[:k]] = I, P[perm[k:]] = C^T; indices = perm[:k].
int id_from_qr(int64_t m, int k, const int64_t* perm, const double* R, int64_t ldr, double* P, int64_t* indices,
               int* warn, cudaStream_t s) {
  Arena ar(s);
  std::vector<double> hr((size_t)k * k);
  SPB_CUDA(cudaMemcpy2DAsync(hr.data(), k * sizeof(double), R, ldr * sizeof(double), k * sizeof(double), k,
                             cudaMemcpyDeviceToHost, s));
  SPB_CUDA(cudaStreamSynchronize(s));
  double dmax = 0.0, dmin = INFINITY;
  for (int i = 0; i < k; ++i) {
    dmax = std::max(dmax, std::fabs(hr[(size_t)i * k + i]));
    dmin = std::min(dmin, std::fabs(hr[(size_t)i * k + i]));
  }
  const int64_t nrest = m - k;
  SPB_ALLOC(ar, double, coef, (size_t)k * std::max<int64_t>(nrest, 1));
  *warn = 0;
  if (nrest > 0) {
    if (dmin > kRankTol * std::max(dmax, 2.2250738585072014e-308)) {
      SPB_TRY(trsm_upper(k, R, ldr, nrest, R + k, ldr, coef, nrest, s));
    } else {
      *warn = SP_WARN_ID_PINV;
      // coef = V diag(pinv(s)) (U^T r2)
      SPB_ALLOC(ar, double, Uu, (size_t)k * k);
      SPB_ALLOC(ar, double, Ss, (size_t)k);
      SPB_ALLOC(ar, double, Vv, (size_t)k * k);
      SPB_ALLOC(ar, double, Si, (size_t)k);
      SPB_ALLOC(ar, double, T, (size_t)k * nrest);
      SPB_ALLOC(ar, double, R1, (size_t)k * k);
      SPB_TRY(copy2d(k, k, R, ldr, R1, k, s));
      SPB_TRY(thin_svd(k, k, R1, k, Uu, k, Ss, Vv, k, s));
      SPB_TRY(pinv_apply(Ss, k, kRankTol, Si, s));
      SPB_TRY(gemm(1, 0, k, nrest, k, 1.0, Uu, k, R + k, ldr, 0.0, T, nrest, s));
      // coef = (V diag(Si)) T
      SPB_TRY(scale_cols(k, k, Vv, k, Si, s));
      SPB_TRY(gemm(0, 0, k, nrest, k, 1.0, Vv, k, T, nrest, 0.0, coef, nrest, s));
    }
  } else if (!(dmin > kRankTol * std::max(dmax, 2.2250738585072014e-308))) {
    *warn = SP_WARN_ID_PINV;
  }
  scatter_p_kernel<<<ceil_div(m * k, 256), 256, 0, s>>>(m, k, perm, coef, std::max<int64_t>(nrest, 1), P);
  count_launch();
  SPB_CHECK_LAUNCH();
  SPB_CUDA(cudaMemcpyAsync(indices, perm, k * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  return SP_OK;
}

// row_id (src/rowid.py:53-79) of M (m x cols): P (m x k), indices (k).
int row_id(int64_t m, int64_t cols, const double* M, int64_t ldm, int k, double* P, int64_t* indices,
           int* warn, cudaStream_t s) {
  SPB_REQUIRE(k >= 1 && k <= std::min(m, cols),
              "rank k=" + std::to_string(k) + " outside [1, " + std::to_string(std::min(m, cols)) + "]");
  Arena ar(s);
  SPB_ALLOC(ar, int64_t, perm, (size_t)m);
  SPB_ALLOC(ar, double, Qp, (size_t)cols * k);
  SPB_ALLOC(ar, double, R, (size_t)k * m);
  // pivoted_qr(M^T): rows = cols of M, candidate columns = rows of M (contiguous)
  SPB_TRY(pivoted_qr(cols, m, M, ldm, k, perm, Qp, k, R, m, s));
  return id_from_qr(m, k, perm, R, m, P, indices, warn, s);
}

// ------------------------------------------------------------ power_id ----
int power_id(const void* A, int a_dtype, int64_t m, int64_t n, int64_t lda, const int64_t* idx,
             const double* w, int depth, int64_t nc, const int64_t* cols, int64_t ncols, int q, int k,
             int r_req, const double* proj, int64_t proj_ell, int id_on_basis, const double* pre_s0,
             const double* pre_c, double* P, int64_t* indices, double* skeleton, double* lift_left,
             double* lift_right, double* lift_ur, int r_max, int64_t* info, cudaStream_t s) {
  const int64_t l0 = launches();
  SPB_REQUIRE(k <= nc, "target rank k=" + std::to_string(k) + " exceeds sketch width n_c=" + std::to_string(nc));
  if (q > 0 || cols) {
    SPB_REQUIRE(cols != nullptr && ncols > 0, "column index set out of range");
    SPB_REQUIRE(ncols > k, "column set size " + std::to_string(ncols) + " must exceed target rank " + std::to_string(k));
    SPB_REQUIRE(ncols >= nc, "column set size " + std::to_string(ncols) + " must cover the sketch width " + std::to_string(nc));
    // with the column block supplied (pre_c: the column-sharded driver's
    // all-gathered C, whose global indices lie outside this shard's n) the
    // indices are not read here; the caller validated them
    if (!pre_c) SPB_TRY(check_columns(cols, ncols, n, s));
  }
  Arena ar(s);
  // coarse sketch (always the plain stencil; projections only feed selection)
  const double* coarse = pre_s0;
  if (!coarse) {
    double* t = ar.alloc<double>((size_t)m * nc);
    if (!t) {
      set_error("sketch allocation failed");
      return SP_ECUDA;
    }
    SPB_TRY(apply_stencil(A, a_dtype, m, n, lda, idx, w, depth, nc, false, t, nc, s));
    coarse = t;
  }
  SPB_TRY(check_finite(m, nc, coarse, nc, "SVD input contains non-finite entries", s));
  // SVD of the coarse sketch: rank and the top-r triplets for the lifting
  const int want = std::max(2 * k, r_req);
  TopSvd top;
  SPB_TRY(svd_top(coarse, m, nc, nc, want, 1.0, top, ar, s, PendingFlag(), /*want_v=*/true, /*need=*/want));
  int rank = top.kept;
  int warn = 0;
  int r = r_req > 0 ? r_req : std::max(k, std::min(2 * k, rank));
  SPB_REQUIRE(r >= k, "lifting rank r=" + std::to_string(r) + " below target rank k=" + std::to_string(k));
  SPB_REQUIRE(r >= 1, "lifting rank r must be >= 1");
  if (r > rank) {
    warn |= SP_WARN_LIFT_CLAMPED;
    r = rank;
  }
  SPB_REQUIRE(r <= top.b && r <= r_max, "lifting rank exceeds the computed basis width");
  // selection input
  const double* sel = coarse;
  int64_t sel_w = nc;
  if (id_on_basis) {
    sel = top.U;  // leading k left singular vectors (ld top.b)
    sel_w = k;
    double* t = ar.alloc<double>((size_t)m * k);
    if (!t) {
      set_error("selection allocation failed");
      return SP_ECUDA;
    }
    SPB_TRY(copy2d(m, k, top.U, top.b, t, k, s));
    sel = t;
  } else if (q > 0) {
    const double* C = pre_c;
    if (!C) {
      double* t = ar.alloc<double>((size_t)m * ncols);
      if (!t) {
        set_error("column block allocation failed");
        return SP_ECUDA;
      }
      SPB_TRY(apply_stencil(A, a_dtype, m, n, lda, cols, nullptr, 1, ncols, true, t, ncols, s));
      C = t;
    }
    double* E = ar.alloc<double>((size_t)m * nc);
    double* E2 = ar.alloc<double>((size_t)m * nc);
    if (ar.failed()) {
      set_error("enriched sketch allocation failed");
      return SP_ECUDA;
    }
    SPB_TRY(copy2d(m, nc, coarse, nc, E, nc, s));
    // C (C^T E) in the reference's association when it is the cheaper one
    // (src/power.py:282-285), each product nearly exactly rounded (Ozaki
    // slices on DMMA, exact_gemm.cu) and the iterate carried in double-double:
    // the greedy pivots past the signal are decided by ulp-level differences
    // of E's residual norms, and only an E this close to the exact product
    // gives the reference's pivots (SPB_ID_PLAIN_GEMM=1: plain FP64 GEMMs).
    // Otherwise (ncols > m, cfg5: C^T C would be 550 GB) W = C C^T, plain FP64.
    const bool ref_order = ncols <= m;
    static const bool plain = getenv("SPB_ID_PLAIN_GEMM") != nullptr;
    double* W = nullptr;
    double *T = nullptr, *T_lo = nullptr, *E_lo = nullptr, *E2_lo = nullptr;
    if (ref_order) {
      T = ar.alloc<double>((size_t)ncols * nc);
      if (!plain) {
        T_lo = ar.alloc<double>((size_t)ncols * nc);
        E_lo = ar.alloc<double>((size_t)m * nc);
        E2_lo = ar.alloc<double>((size_t)m * nc);
      }
    } else {
      W = ar.alloc<double>((size_t)m * m);
    }
    if (ar.failed()) {
      set_error("enriched sketch allocation failed");
      return SP_ECUDA;
    }
    bool sym_t = false;
    if (ref_order && !plain && !proj && ncols == nc && getenv("SPB_ID_FULL_T") == nullptr)
      SPB_TRY(sketch_is_columns(idx, w, depth, nc, nullptr, cols, ncols, sym_t, s));
    if (!ref_order) SPB_TRY(gemm_aat(m, ncols, C, ncols, W, m, s));  // W = C C^T, upper tiles + mirror
    for (int it = 0; it < q; ++it) {
      if (ref_order && plain) {
        SPB_TRY(gemm(1, 0, ncols, nc, m, 1.0, C, ncols, E, nc, 0.0, T, nc, s));
        SPB_TRY(gemm(0, 0, m, nc, ncols, 1.0, C, ncols, T, nc, 0.0, E2, nc, s));
      } else if (ref_order) {
        // first step with the sketch on the same column set: E = s0 = C bit for
        // bit, T = C^T C is symmetric (upper tiles + mirror; SPB_ID_FULL_T=1: all tiles)
        SPB_TRY(gemm_exact(1, ncols, nc, m, C, ncols, E, it == 0 ? nullptr : E_lo, nc, T, T_lo, nc, s,
                           it == 0 && sym_t));
        SPB_TRY(gemm_exact(0, m, nc, ncols, C, ncols, T, T_lo, nc, E2, E2_lo, nc, s));
        std::swap(E_lo, E2_lo);
      } else {
        SPB_TRY(gemm(0, 0, m, nc, m, 1.0, W, m, E, nc, 0.0, E2, nc, s));
      }
      SPB_TRY(check_finite(m, nc, E2, nc, "power iterate overflowed; enable re-orthonormalization (reorth)", s));
      std::swap(E, E2);
    }
    sel = E;
  }
  if (proj && !id_on_basis) {
    double* t = ar.alloc<double>((size_t)m * proj_ell);
    if (!t) {
      set_error("projection allocation failed");
      return SP_ECUDA;
    }
    SPB_TRY(gemm(0, 0, m, proj_ell, sel_w, 1.0, sel, sel_w, proj, proj_ell, 0.0, t, proj_ell, s));
    sel = t;
    sel_w = proj_ell;
  }
  int idwarn = 0;
  SPB_TRY(row_id(m, sel_w, sel, sel_w, k, P, indices, &idwarn, s));
  warn |= idwarn;
  // skeleton = coarse[indices]
  gather_rows_kernel<<<ceil_div((int64_t)k * nc, 256), 256, 0, s>>>(indices, k, coarse, nc, nc, skeleton, nc);
  count_launch();
  SPB_CHECK_LAUNCH();
  // lifting T = (V_r S_r^{-1}) (U_r^T A), kept factored
  if (r > 0) {
    SPB_ALLOC(ar, double, sinv, (size_t)top.b);
    SPB_TRY(pinv_apply(top.S, top.b, kRankTol, sinv, s));
    SPB_TRY(copy2d(nc, r, top.V, top.b, lift_left, r_max, s));
    SPB_TRY(scale_cols(nc, r, lift_left, r_max, sinv, s));
    if (lift_ur) SPB_TRY(copy2d(m, r, top.U, top.b, lift_ur, r_max, s));
    if (lift_right && a_dtype == SP_F64) {
      SPB_TRY(gemm(1, 0, r, n, m, 1.0, top.U, top.b, (const double*)A, lda, 0.0, lift_right, n, s));
    } else if (lift_right) {
      // Y = A^T U_r (n x r) with FP32 A (16-column slabs), then transpose
      SPB_ALLOC(ar, double, Yt, (size_t)n * r);
      SPB_TRY(skinny_atz(A, a_dtype, m, n, lda, top.U, top.b, r, Yt, r, s));
      SPB_TRY(transpose(n, r, Yt, r, lift_right, n, s));
    }
  }
  if (top.bulk) warn |= SP_WARN_BULK_SPLIT;
  if (info) {
    fill_info(info, r, warn, top, l0);
    info[SP_INFO_RANK] = rank;
    info[SP_INFO_LIFT_R] = r;
  }
  return SP_OK;
}

}  // namespace spb
