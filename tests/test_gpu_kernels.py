"""GPU kernel-level parity: each C-ABI entry point against the oracle / numpy.

Bit-exact gates for the gather (K1) and the pivot order (K7); the floating
point kernels against a numpy FP64 reference with the tolerance written in
each test.  All calls go through the C-ABI (ctypes) of libsketchpress_b200.so.
"""

import numpy as np
import pytest

from conftest import load_golden, philox, rank_deficient

import oracle
import paper_2105_01271_b200 as sp
from paper_2105_01271_b200 import _lib

pytestmark = pytest.mark.gpu


def _dev(x, cuda):
    return cuda.from_numpy(np.ascontiguousarray(x)).cuda()


def _stream(cuda):
    return cuda.cuda.current_stream().cuda_stream


# ------------------------------------------------------------------ K1 ----
@pytest.mark.parametrize("kind", ["injection", "neighbor", "global"])
@pytest.mark.parametrize("n,n_c", [(37, 9), (4096, 256), (1000, 999), (50, 3)])
def test_stencil_bit_exact(cuda, kind, n, n_c):
    x = philox(n + n_c).standard_normal((70, n))
    x[3, :5] = -0.0
    op = sp.build_sketch(sp.SketchSpec(kind, n, n_c))
    got = sp.apply_sketch(op, x)
    want = oracle.sketch_rows(x, op.idx, op.w)
    assert got.shape == want.shape
    assert np.array_equal(got, want)  # == : -0.0 becomes +0.0 in both


def test_stencil_golden_tables(cuda):
    g = load_golden("small_cases.npz")
    x = philox(21).standard_normal((5, 37))
    for kind in ("injection", "neighbor", "global"):
        op = sp.build_sketch(sp.SketchSpec(kind, 37, 9))
        assert np.array_equal(op.idx, g[f"st_{kind}_idx"])
        assert np.array_equal(op.w, g[f"st_{kind}_w"])
        assert np.array_equal(sp.apply_sketch(op, x), g[f"st_{kind}_out"])


def test_gather_columns_exact_and_f32(cuda):
    x = philox(3).standard_normal((33, 500))
    cols = np.array([0, 7, 499, 250, 3])
    assert np.array_equal(sp.gather_columns(x, cols), x[:, cols])
    xf = x.astype(np.float32)
    d = _dev(xf, cuda)
    out = sp.gather_columns(d, cols).cpu().numpy()
    assert np.array_equal(out, xf[:, cols].astype(np.float64))
    with pytest.raises(sp.ConfigError):
        sp.gather_columns(x, [1, 1])
    with pytest.raises(sp.ConfigError):
        sp.gather_columns(x, [500])


def test_grid_injection_indices_bit_exact(cuda):
    op, cols = sp.grid_injection((64, 64), 4)
    assert np.array_equal(cols, oracle.grid_coarse_indices((64, 64), 4))
    op3, cols3 = sp.grid_injection((16, 12, 8), 4)
    want = np.array([(ix * 12 + iy) * 8 + iz for ix in range(0, 16, 4) for iy in range(0, 12, 4)
                     for iz in range(0, 8, 4)])
    assert np.array_equal(cols3, want)


# ------------------------------------------------------------------ K2 ----
@pytest.mark.parametrize("r", [1, 3, 7, 8, 16, 24, 32])
@pytest.mark.parametrize("m,n", [(1000, 4096), (257, 1001), (5, 33), (5, 34), (3, 4096), (2001, 20002)])
def test_skinny_atz(cuda, r, m, n):
    rng = philox(m * r + n)
    a = rng.standard_normal((m, n))
    z = rng.standard_normal((m, r))
    y = cuda.empty((n, r), dtype=cuda.float64, device="cuda")
    da, dz = _dev(a, cuda), _dev(z, cuda)
    _lib.call("sp_skinny_atz", da.data_ptr(), _lib.SP_F64, m, n, n, dz.data_ptr(), r, r, y.data_ptr(), r,
              _stream(cuda))
    want = a.T @ z
    np.testing.assert_allclose(y.cpu().numpy(), want, rtol=0, atol=1e-12 * np.abs(a).sum(0).max() * np.abs(z).max())


def test_skinny_atz_f32_and_determinism(cuda):
    rng = philox(5)
    a = rng.standard_normal((600, 3000)).astype(np.float32)
    z = rng.standard_normal((600, 8))
    da, dz = _dev(a, cuda), _dev(z, cuda)
    outs = []
    for _ in range(2):
        y = cuda.empty((3000, 8), dtype=cuda.float64, device="cuda")
        _lib.call("sp_skinny_atz", da.data_ptr(), _lib.SP_F32, 600, 3000, 3000, dz.data_ptr(), 8, 8,
                  y.data_ptr(), 8, _stream(cuda))
        outs.append(y.cpu().numpy())
    # f32 x f64 products are exact in f64: only the sums round
    np.testing.assert_allclose(outs[0], a.astype(np.float64).T @ z, rtol=0, atol=1e-11)
    assert outs[0].tobytes() == outs[1].tobytes()  # fixed reduction order


# ------------------------------------------------------------------ K3 ----
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(64, 64, 16), (100, 37, 259), (3, 200, 4000), (513, 65, 7),
                                   (7, 7, 65536), (40, 33, 3000), (64, 64, 5000), (2, 3, 700),
                                   (3000, 33, 40), (5000, 64, 64), (700, 1, 1), (65536, 43, 7),
                                   (2000, 32, 4096), (4096, 32, 2000), (130, 5, 300), (129, 31, 70),
                                   (70000, 5, 5), (70000, 16, 3), (9000, 200, 5), (5000, 100, 64)])
def test_gemm(cuda, ta, tb, M, N, K):
    rng = philox(M + N + K + ta * 2 + tb)
    A = rng.standard_normal((K, M) if ta else (M, K))
    B = rng.standard_normal((N, K) if tb else (K, N))
    C0 = rng.standard_normal((M, N))
    dA, dB, dC = _dev(A, cuda), _dev(B, cuda), _dev(C0, cuda)
    _lib.call("sp_gemm", ta, tb, M, N, K, 1.5, dA.data_ptr(), A.shape[1], dB.data_ptr(), B.shape[1], -0.5,
              dC.data_ptr(), N, _stream(cuda))
    want = 1.5 * (A.T if ta else A) @ (B.T if tb else B) - 0.5 * C0
    np.testing.assert_allclose(dC.cpu().numpy(), want, rtol=0, atol=1e-12 * np.sqrt(K) * 8)


@pytest.mark.parametrize("M,K", [(1, 5), (64, 300), (65, 300), (200, 1000), (333, 4100), (2000, 9000)])
def test_gemm_aat_symmetric_product(cuda, M, K):
    """W = A A^T from the upper tiles + mirror equals the plain product and is
    exactly symmetric (src/power.py:99-108 in the (C C^T) s0 association)."""
    A = philox(M + K).standard_normal((M, K))
    dA = _dev(A, cuda)
    W = cuda.full((M, M), float("nan"), dtype=cuda.float64, device="cuda")
    _lib.call("sp_gemm_aat", M, K, dA.data_ptr(), K, W.data_ptr(), M, _stream(cuda))
    w = W.cpu().numpy()
    np.testing.assert_array_equal(w, w.T)
    np.testing.assert_allclose(w, A @ A.T, rtol=0, atol=1e-12 * np.sqrt(K) * 8)


@pytest.mark.parametrize("M,N,K", [(300, 1, 64), (300, 2, 64), (1000, 3, 64), (257, 4, 63), (4096, 4, 64)])
def test_gemm_tall_times_narrow(cuda, M, N, K):
    """Tall X (M x K <= 64) times a narrow block (N <= 4): the row-tile kernel's
    shared-memory request is bounded by the opt-in (it asked for 268 KB and the
    launch failed; found by scripts/fuzz_api.py), and a failed launch no longer
    leaves its error behind for the next call."""
    rng = philox(M + N + K)
    A, B = rng.standard_normal((M, K)), rng.standard_normal((K, N))
    dA, dB = _dev(A, cuda), _dev(B, cuda)
    dC = cuda.zeros((M, N), dtype=cuda.float64, device="cuda")
    _lib.call("sp_gemm", 0, 0, M, N, K, 1.0, dA.data_ptr(), K, dB.data_ptr(), N, 0.0, dC.data_ptr(), N, _stream(cuda))
    np.testing.assert_allclose(dC.cpu().numpy(), A @ B, rtol=0, atol=1e-12)


# ------------------------------------------------------------------ K4 ----
@pytest.mark.parametrize("rows,cols", [(1000, 8), (5000, 32), (70000, 20), (300, 64), (2000, 100), (32, 32),
                                       (4096, 32), (65536, 7), (257, 32), (33, 32), (512, 1), (100, 3),
                                       (200000, 32), (7, 7), (4097, 32), (5120, 32), (5121, 32), (4800, 17),
                                       (5000, 216)])
def test_tsqr(cuda, rows, cols):
    x = philox(rows + cols).standard_normal((rows, cols)) * np.logspace(0, -8, cols)
    dx = _dev(x, cuda)
    q = cuda.empty((rows, cols), dtype=cuda.float64, device="cuda")
    r = cuda.empty((cols, cols), dtype=cuda.float64, device="cuda")
    _lib.call("sp_tsqr", rows, cols, dx.data_ptr(), cols, q.data_ptr(), cols, r.data_ptr(), cols, _stream(cuda))
    q, r = q.cpu().numpy(), r.cpu().numpy()
    assert np.abs(q.T @ q - np.eye(cols)).max() < 1e-13
    assert np.linalg.norm(q @ r - x) <= 1e-14 * np.linalg.norm(x) * np.sqrt(rows)
    assert np.allclose(np.tril(r, -1), 0)
    assert np.all(np.diag(r) >= 0)


@pytest.mark.parametrize("rows,cols,cond", [(65536, 7, 1e4), (2000, 50, 10.0), (300, 64, 1e5), (5000, 112, 1e3)])
def test_cholqr2_well_conditioned(cuda, rows, cols, cond):
    x = philox(rows + cols).standard_normal((rows, cols)) * np.logspace(0, -np.log10(cond), cols)
    dx = _dev(x, cuda)
    q = cuda.empty((rows, cols), dtype=cuda.float64, device="cuda")
    r = cuda.empty((cols, cols), dtype=cuda.float64, device="cuda")
    _lib.call("sp_qr_tall", rows, cols, dx.data_ptr(), cols, q.data_ptr(), cols, r.data_ptr(), cols, 1,
              _stream(cuda))
    q, r = q.cpu().numpy(), r.cpu().numpy()
    assert np.abs(q.T @ q - np.eye(cols)).max() < 1e-13
    assert np.linalg.norm(q @ r - x) <= 1e-14 * np.linalg.norm(x) * np.sqrt(cols)
    assert np.allclose(np.tril(r, -1), 0) and np.all(np.diag(r) > 0)


def test_cholqr2_breakdown_falls_back(cuda):
    x = rank_deficient(philox(9), 2000, 20, 4)
    dx = _dev(x, cuda)
    q = cuda.empty((2000, 20), dtype=cuda.float64, device="cuda")
    r = cuda.empty((20, 20), dtype=cuda.float64, device="cuda")
    _lib.call("sp_qr_tall", 2000, 20, dx.data_ptr(), 20, q.data_ptr(), 20, r.data_ptr(), 20, 1, _stream(cuda))
    q, r = q.cpu().numpy(), r.cpu().numpy()
    assert np.abs(q.T @ q - np.eye(20)).max() < 1e-12
    assert np.linalg.norm(q @ r - x) <= 1e-13 * np.linalg.norm(x)


@pytest.mark.parametrize("rows,cols,rank", [(4096, 32, 9), (2000, 32, 1), (65536, 7, 3), (300, 20, 0),
                                            (1000, 256, 10), (4096, 100, 3)])
def test_tsqr32_rank_deficient(cuda, rows, cols, rank):
    x = rank_deficient(philox(rows + rank), rows, cols, rank) if rank else np.zeros((rows, cols))
    if rank:
        x[:, 3] = 0.0  # an exactly zero column
    dx = _dev(x, cuda)
    q = cuda.empty((rows, cols), dtype=cuda.float64, device="cuda")
    r = cuda.empty((cols, cols), dtype=cuda.float64, device="cuda")
    for _ in range(2):
        _lib.call("sp_tsqr", rows, cols, dx.data_ptr(), cols, q.data_ptr(), cols, r.data_ptr(), cols,
                  _stream(cuda))
        qn, rn = q.cpu().numpy(), r.cpu().numpy()
        assert np.abs(qn.T @ qn - np.eye(cols)).max() < 1e-12
        assert np.linalg.norm(qn @ rn - x) <= 1e-13 * max(np.linalg.norm(x), 1e-300)
        assert np.allclose(np.tril(rn, -1), 0) and np.all(np.diag(rn) >= 0)
        if _ == 0:
            first = (qn.tobytes(), rn.tobytes())
    assert (qn.tobytes(), rn.tobytes()) == first  # bitwise reproducible


def test_tsqr_rank_deficient_keeps_orthonormality(cuda):
    x = rank_deficient(philox(4), 3000, 40, 5)
    dx = _dev(x, cuda)
    q = cuda.empty((3000, 40), dtype=cuda.float64, device="cuda")
    r = cuda.empty((40, 40), dtype=cuda.float64, device="cuda")
    _lib.call("sp_tsqr", 3000, 40, dx.data_ptr(), 40, q.data_ptr(), 40, r.data_ptr(), 40, _stream(cuda))
    q, r = q.cpu().numpy(), r.cpu().numpy()
    assert np.abs(q.T @ q - np.eye(40)).max() < 1e-12
    assert np.linalg.norm(q @ r - x) <= 1e-13 * np.linalg.norm(x)


# ------------------------------------------------------------------ K5 ----
@pytest.mark.parametrize("n", [1, 2, 7, 32, 64, 113, 120, 200, 256])
def test_jacobi_svd(cuda, n):
    rng = philox(n)
    m = rng.standard_normal((n, n)) @ np.diag(np.logspace(0, -10, n))
    dm = _dev(m, cuda)
    u = cuda.zeros((n, n), dtype=cuda.float64, device="cuda")
    s = cuda.zeros((n,), dtype=cuda.float64, device="cuda")
    v = cuda.zeros((n, n), dtype=cuda.float64, device="cuda")
    _lib.call("sp_jacobi_svd", n, dm.data_ptr(), n, u.data_ptr(), n, s.data_ptr(), v.data_ptr(), n, _stream(cuda))
    u, s, v = u.cpu().numpy(), s.cpu().numpy(), v.cpu().numpy()
    want = np.linalg.svd(m, compute_uv=False)
    assert np.all(np.diff(s) <= 0)
    np.testing.assert_allclose(s, want, rtol=1e-12 * n, atol=1e-15 * want[0] * n)
    np.testing.assert_allclose((u * s) @ v.T, m, atol=1e-14 * want[0] * n)
    np.testing.assert_allclose(v.T @ v, np.eye(n), atol=1e-13)


@pytest.mark.parametrize("shape,rank", [((300, 48), 16), ((17, 64), 5), ((33, 2), 1), ((5200, 256), 85),
                                        ((17, 216), 5), ((64, 64), 0), ((40, 40), 39)])
def test_thin_svd_rank_deficient_small_core_is_orthonormal(cuda, shape, rank):
    """Exact zeros in the spectrum with a core of <= 256 columns: U and V stay
    orthonormal (LAPACK completes the null directions, src/kernels.py:87-94); the
    normalised Jacobi columns are rounding noise there (found by scripts/fuzz_dense.py)."""
    rows, cols = shape
    p = min(rows, cols)
    m = rank_deficient(philox(rows + cols), rows, cols, rank) if rank else np.zeros(shape)
    f = sp.thin_svd(m)
    s_ref = np.linalg.svd(m, compute_uv=False)
    np.testing.assert_allclose(f.s, s_ref, rtol=0, atol=1e-13 * max(s_ref[0], 1.0))
    np.testing.assert_allclose(f.u.T @ f.u, np.eye(p), atol=1e-11)
    np.testing.assert_allclose(f.v.T @ f.v, np.eye(p), atol=1e-11)
    np.testing.assert_allclose((f.u * f.s) @ f.v.T, m, atol=1e-12 * max(s_ref[0], 1.0))


@pytest.mark.parametrize("n", [24, 32, 48, 96, 200, 256, 300])
def test_jacobi_svd_flat_spectrum_stays_orthonormal(cuda, n):
    """A flat stretch of (nearly) equal singular values: the rotations inside the
    cluster are large-angle however small the couplings, so the quadratic-
    convergence stop alone left 2-4e-9 of non-orthogonality in U (found by
    scripts/fuzz_api.py); a sweep with a large-angle rotation is the last only once its
    couplings are below 1e-11."""
    rng = philox(700 + n)
    s_true = np.r_[np.logspace(0, -2, 6), np.full(n - 6, 3e-3)]
    q1, _ = np.linalg.qr(rng.standard_normal((n, n)))
    q2, _ = np.linalg.qr(rng.standard_normal((n, n)))
    m = (q1 * s_true) @ q2.T
    f = sp.thin_svd(m)
    np.testing.assert_allclose(f.s, np.sort(s_true)[::-1], rtol=0, atol=1e-14)
    np.testing.assert_allclose(f.u.T @ f.u, np.eye(n), atol=5e-11)
    np.testing.assert_allclose(f.v.T @ f.v, np.eye(n), atol=5e-11)
    np.testing.assert_allclose((f.u * f.s) @ f.v.T, m, atol=1e-13)


@pytest.mark.parametrize("n,decay", [(3, 0.0), (16, -14.0), (31, -3.0), (32, -16.0), (32, -30.0)])
def test_jacobi_svd_small_without_v(cuda, n, decay):
    """n <= 32 lane-per-column kernel, U and S only (V not accumulated)."""
    rng = philox(100 + n)
    m = rng.standard_normal((n, n)) @ np.diag(np.logspace(0, decay, n)) @ rng.standard_normal((n, n))
    dm = _dev(m, cuda)
    u = cuda.zeros((n, n), dtype=cuda.float64, device="cuda")
    s = cuda.zeros((n,), dtype=cuda.float64, device="cuda")
    _lib.call("sp_jacobi_svd", n, dm.data_ptr(), n, u.data_ptr(), n, s.data_ptr(), None, n, _stream(cuda))
    u, s = u.cpu().numpy(), s.cpu().numpy()
    want = np.linalg.svd(m, compute_uv=False)
    assert np.all(np.diff(s) <= 0)
    np.testing.assert_allclose(s, want, rtol=0, atol=1e-14 * want[0] * n)
    keep = s > 1e-8 * s[0]  # well separated, well above rounding: unique up to sign
    uref = np.linalg.svd(m)[0][:, keep]
    np.testing.assert_allclose(np.abs(np.sum(u[:, keep] * uref, axis=0)), 1.0, atol=1e-9)


# ------------------------------------------------------ API dense kernels ----
@pytest.mark.parametrize("shape", [(5, 7), (7, 5), (20, 11), (50, 80), (80, 50), (3000, 40)])
def test_thin_qr_matches_reference_convention(cuda, shape):
    m = philox(sum(shape)).standard_normal(shape)
    fac = sp.thin_qr(m)
    q_ref, r_ref = oracle.qr_reduced(m)
    # unique for full rank once the sign convention is applied
    np.testing.assert_allclose(fac.q, q_ref, atol=1e-12)
    np.testing.assert_allclose(fac.r, r_ref, atol=1e-12 * np.abs(r_ref).max())


@pytest.mark.parametrize("shape", [(5, 7), (12, 9), (50, 80), (2000, 30)])
def test_thin_svd_matches_reference_convention(cuda, shape):
    m = philox(shape[0]).standard_normal(shape)
    fac = sp.thin_svd(m)
    u_ref, s_ref, v_ref = oracle.svd_thin(m)
    np.testing.assert_allclose(fac.s, s_ref, rtol=1e-13)
    np.testing.assert_allclose(fac.u, u_ref, atol=1e-11)
    np.testing.assert_allclose(fac.v, v_ref, atol=1e-11)


def test_pinv_apply(cuda):
    np.testing.assert_allclose(sp.pinv_apply(np.array([2.0, 1.0, 0.0])), [0.5, 1.0, 0.0])
    np.testing.assert_allclose(sp.pinv_apply(np.array([1.0, 1e-18])), [1.0, 0.0])
    np.testing.assert_array_equal(sp.pinv_apply(np.zeros(3)), np.zeros(3))
    with pytest.raises(sp.ConfigError):
        sp.pinv_apply(np.array([1.0, 2.0]))


# ------------------------------------------------------------------ K7 ----
def test_pivoted_qr_golden_and_oracle(cuda):
    g = load_golden("small_cases.npz")
    m = philox(12).standard_normal((10, 8)) * np.logspace(0, -3, 8)
    f = sp.pivoted_qr(m, 6)
    assert np.array_equal(f.perm, g["pq_perm"])
    np.testing.assert_allclose(f.r, g["pq_r"], atol=1e-13)
    np.testing.assert_allclose(f.q, g["pq_q"], atol=1e-13)


def test_pivoted_qr_duplicate_columns_tie_break(cuda):
    base = philox(10).standard_normal(4)
    m = np.column_stack([base, base, 2.0 * base, base])
    fac = sp.pivoted_qr(m, 2)
    assert fac.perm[0] == 2 and fac.perm[1] == 0


@pytest.mark.parametrize("rows,cols,k", [(64, 300, 40), (200, 1000, 100), (9, 6, 6),
                                        (40000, 300, 60), (70000, 64, 64),
                                        # register-resident update: 1025 .. 4096 rows, ragged and full
                                        (1025, 700, 50), (2048, 500, 64), (3000, 900, 80), (4096, 1200, 100),
                                        (4097, 300, 40),
                                        # very long candidates (the row-block path), ragged
                                        (140000, 40, 20), (262144, 24, 24), (200001, 33, 10)])
def test_pivoted_qr_matches_oracle_pivots(cuda, rows, cols, k):
    m = philox(rows * cols).standard_normal((rows, cols)) * np.logspace(0, -2, cols)
    f = sp.pivoted_qr(m, k)
    q_o, r_o, perm_o = oracle.greedy_pivoted_qr(m, k)
    gaps = oracle.pivot_gaps(m, k)
    pstar = k if np.all(gaps > 1e-11) else int(np.argmax(gaps <= 1e-11))
    assert np.array_equal(f.perm[:pstar], perm_o[:pstar])
    np.testing.assert_allclose(f.q @ f.r, m[:, f.perm], atol=1e-10 * np.linalg.norm(m)) if k == min(rows, cols) else None


def test_pivoted_qr_long_candidates_rank_deficient(cuda):
    """Long candidates (the row-block path) with an exact zero residual:
    falls back to the per-candidate path and its deterministic filler."""
    rng = philox(77)
    base = rng.standard_normal((40000, 3))
    m = np.column_stack([base, base @ rng.standard_normal((3, 5))])  # rank 3, 8 candidates
    f = sp.pivoted_qr(m, 6)
    np.testing.assert_allclose(f.q.T @ f.q, np.eye(6), atol=1e-12)
    q_o, r_o, perm_o = oracle.greedy_pivoted_qr(m, 6)
    assert np.array_equal(f.perm[:3], perm_o[:3])


def test_row_id_golden(cuda):
    g = load_golden("small_cases.npz")
    m = philox(1).standard_normal((9, 5))
    f = sp.row_id(m, 3)
    assert np.array_equal(f.indices, g["rid_idx"])
    np.testing.assert_allclose(f.p, g["rid_p"], atol=1e-12)
    np.testing.assert_array_equal(f.p[f.indices], np.eye(3))
    h = sp.row_id(np.array([[1.0, 2.0], [2.0, 4.0]]), 1)
    np.testing.assert_array_equal(h.indices, [1])
    np.testing.assert_allclose(h.p, [[0.5], [1.0]])


@pytest.mark.parametrize("N,r,k", [(2000, 7, 50), (65536, 7, 50), (5000, 5, 200), (300, 1, 64),
                                   (1000, 20, 220), (500, 32, 96)])
def test_householder_complete(cuda, N, r, k):
    """Columns [r, k) become an orthonormal completion of the orthonormal
    columns [0, r) (Householder reconstruction, sp_householder_complete)."""
    q, _ = np.linalg.qr(philox(N + r + k).standard_normal((N, r)))
    out = np.zeros((N, k))
    out[:, :r] = q
    d = _dev(out, cuda)
    kp = cuda.empty((r, k - r), dtype=cuda.float64, device="cuda")
    _lib.call("sp_householder_complete", N, r, k, d.data_ptr(), k, kp.data_ptr(), _stream(cuda))
    o = d.cpu().numpy()
    np.testing.assert_array_equal(o[:, :r], q)  # untouched
    np.testing.assert_allclose(o.T @ o, np.eye(k), atol=1e-13)


@pytest.mark.parametrize("m,n,k,f32", [(300, 1000, 7, False), (257, 700, 64, False), (100, 333, 200, False),
                                       (120, 500, 20, True)])
def test_frob_residual(cuda, m, n, k, f32):
    """K8: ||A - U diag(S) V^T||_F^2 and ||A||_F^2 without forming U S V^T."""
    rng = philox(m + n + k)
    a = rng.standard_normal((m, n))
    if f32:
        a = a.astype(np.float32)
    u, s, v = rng.standard_normal((m, k)), rng.random(k), rng.standard_normal((n, k))
    out = np.zeros(2)
    da = cuda.from_numpy(a).cuda()
    du, ds, dv = _dev(u, cuda), _dev(s, cuda), _dev(v, cuda)
    _lib.call("sp_frob_residual", da.data_ptr(), _lib.SP_F32 if f32 else _lib.SP_F64, m, n, n, du.data_ptr(), k,
              ds.data_ptr(), dv.data_ptr(), k, k, out.ctypes.data_as(__import__("ctypes").c_void_p), _stream(cuda))
    a64 = a.astype(np.float64)
    want = np.sum((a64 - (u * s) @ v.T) ** 2), np.sum(a64 ** 2)
    np.testing.assert_allclose(out, want, rtol=1e-12)


# ------------------------------------------------------- SRHT test block ----
def _srht(cuda, x, b, seed=7):
    rows, cols = x.shape
    X = _dev(x, cuda)
    Y = cuda.empty((rows, b), dtype=cuda.float64, device="cuda")
    flag = cuda.zeros(1, dtype=cuda.int32, device="cuda")
    _lib.call("sp_srht_sketch", rows, cols, X.data_ptr(), cols, b, seed, Y.data_ptr(), b, flag.data_ptr(),
              _stream(cuda))
    return Y.cpu().numpy(), int(flag.item())


@pytest.mark.parametrize("cols,b", [(256, 32), (300, 32), (1000, 16), (4096, 32), (4096, 16), (5000, 32),
                                    (16384, 32)])
def test_srht_is_a_scaled_orthogonal_sampling(cuda, cols, b):
    # Omega = D H S (one row per basis vector): Omega^T Omega = N I_b exactly
    # (distinct Hadamard columns of the padded width N), and Y(X) = X Omega.
    n2 = 256
    while n2 < cols:
        n2 *= 2
    x = philox(cols + b).standard_normal((37, cols))
    y, _ = _srht(cuda, x, b)
    if cols > 5000:  # explicit Omega too large: linearity and the scale of H
        x2 = philox(cols + 2 * b).standard_normal((37, cols))
        y2, _ = _srht(cuda, x2, b)
        y12, _ = _srht(cuda, x + x2, b)
        np.testing.assert_allclose(y12, y + y2, rtol=0, atol=1e-11 * np.sqrt(cols) * 40)
        return
    eye = np.eye(cols)
    om, flag = _srht(cuda, eye, b)
    assert flag == 0
    assert set(np.unique(np.abs(om))) <= {1.0}  # +-1 entries
    if cols == n2:  # unpadded width: the sampled Hadamard columns are exactly orthogonal
        np.testing.assert_array_equal(om.T @ om, n2 * np.eye(b))
    else:  # padded to the next power of two: still full column rank
        assert np.linalg.matrix_rank(om) == b
    np.testing.assert_allclose(y, x @ om, rtol=0, atol=1e-13 * np.abs(x).sum(axis=1).max())
    # deterministic: bitwise identical on a second call
    y2, _ = _srht(cuda, x, b)
    assert np.array_equal(y, y2)


def test_srht_flags_non_finite_input(cuda):
    x = philox(3).standard_normal((10, 700))
    x[4, 123] = np.nan
    _, flag = _srht(cuda, x, 32)
    assert flag == 1


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_srht_gather_is_exact_and_matches_two_step(cuda, dtype):
    a = philox(11).standard_normal((130, 9000))
    if dtype == "f32":
        a = a.astype(np.float32)
    a[5, 17] = -0.0
    idx = np.sort(philox(12).choice(9000, size=4000, replace=False)).astype(np.int64)
    A = _dev(a, cuda)
    I = _dev(idx, cuda)
    X = cuda.empty((130, idx.size), dtype=cuda.float64, device="cuda")
    Y = cuda.empty((130, 32), dtype=cuda.float64, device="cuda")
    flag = cuda.zeros(1, dtype=cuda.int32, device="cuda")
    tag = _lib.SP_F64 if dtype == "f64" else _lib.SP_F32
    _lib.call("sp_srht_gather", A.data_ptr(), tag, 130, 9000, I.data_ptr(), idx.size, X.data_ptr(), idx.size, 32, 99,
              Y.data_ptr(), 32, flag.data_ptr(), _stream(cuda))
    xg = X.cpu().numpy()
    want = a[:, idx].astype(np.float64)
    assert np.array_equal(xg.view(np.int64), want.view(np.int64))  # bit-exact copies, -0.0 kept
    y2, f2 = _srht(cuda, want, 32, seed=99)
    assert np.array_equal(Y.cpu().numpy(), y2) and int(flag.item()) == 0 and f2 == 0


def _srht_gather(cuda, a, idx, b=32, seed=99):
    rows, n = a.shape
    A, I = _dev(a, cuda), _dev(idx, cuda)
    X = cuda.empty((rows, idx.size), dtype=cuda.float64, device="cuda")
    Y = cuda.empty((rows, b), dtype=cuda.float64, device="cuda")
    flag = cuda.zeros(1, dtype=cuda.int32, device="cuda")
    tag = _lib.SP_F64 if a.dtype == np.float64 else _lib.SP_F32
    _lib.call("sp_srht_gather", A.data_ptr(), tag, rows, n, I.data_ptr(), idx.size, X.data_ptr(), idx.size, b, seed,
              Y.data_ptr(), b, flag.data_ptr(), _stream(cuda))
    return X.cpu().numpy(), Y.cpu().numpy(), int(flag.item())


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_srht_gather_chunked_rows(cuda, dtype):
    # rows wider than 16384 gathered columns (cfg5: 262144): 16384-column
    # chunks with their own signs and the same samples, summed in chunk order
    rows, n, nc = 70, 60000, 40000  # chunks of 16384, 16384, 7232
    a = philox(21).standard_normal((rows, n))
    if dtype == "f32":
        a = a.astype(np.float32)
    idx = np.sort(philox(22).choice(n, size=nc, replace=False)).astype(np.int64)
    x, y, flag = _srht_gather(cuda, a, idx)
    want = a[:, idx].astype(np.float64)
    assert flag == 0
    assert np.array_equal(x.view(np.int64), want.view(np.int64))
    # chunk 0 alone is the plain 16384-wide transform with the same seed
    a0 = np.zeros_like(a)
    a0[:, idx[:16384]] = a[:, idx[:16384]]
    _, y0, _ = _srht_gather(cuda, a0, idx)
    y0_ref, _ = _srht(cuda, want[:, :16384], 32, seed=99)
    assert np.array_equal(y0, y0_ref)
    # a single entry in chunk 2: +-value at every sample (Hadamard entries are
    # +-1), and linearity over the chunks (sum of the per-chunk test blocks)
    e = np.zeros_like(a)
    e[3, idx[33000]] = 0.75
    _, ye, _ = _srht_gather(cuda, e, idx)
    assert np.all(np.abs(ye[3]) == 0.75) and np.all(np.delete(ye, 3, axis=0) == 0.0)
    a1, a2 = a0, a - a0
    _, y1, _ = _srht_gather(cuda, a1, idx)
    _, y2, _ = _srht_gather(cuda, a2, idx)
    np.testing.assert_allclose(y, y1 + y2, rtol=0, atol=1e-12 * np.abs(y).max())
    # the chunks' sign patterns differ: the same local position in chunk 1
    # gives a different row of Omega than in chunk 0
    e0 = np.zeros_like(a)
    e0[0, idx[100]] = 1.0
    e0[1, idx[16384 + 100]] = 1.0
    _, yd, _ = _srht_gather(cuda, e0, idx)
    assert np.all(np.abs(yd[:2]) == 1.0) and not np.array_equal(yd[0], yd[1])


# ------------------------------------------------- double-double Gram R ----
def _gram_chol_dd(cuda, x):
    rows, b = x.shape
    X = _dev(x, cuda)
    R = cuda.full((b, b), float("nan"), dtype=cuda.float64, device="cuda")
    _lib.call("sp_gram_chol_dd", rows, b, X.data_ptr(), b, R.data_ptr(), b, _stream(cuda))
    return R.cpu().numpy()


@pytest.mark.parametrize("rows,b,decay", [(4096, 32, 0.3), (2000, 32, 0.1), (700, 20, 0.5), (262144, 32, 0.35),
                                          (64, 32, 0.6), (33, 7, 0.9)])
def test_gram_chol_dd_matches_householder_r(cuda, rows, b, decay):
    # graded singular values down to ~1e-17 of the largest (a numerically
    # rank-deficient subspace block): R must be upper triangular with a
    # non-negative diagonal, R^T R = X^T X to dd-rounded FP64, and the
    # singular values of R must match the Householder R's (LAPACK) to ~1e-15
    # of the largest; the top singular subspace of R^T must match too.
    rng = philox(rows + 31 * b)
    u, _ = np.linalg.qr(rng.standard_normal((rows, b)))
    v, _ = np.linalg.qr(rng.standard_normal((b, b)))
    sv = np.maximum(decay ** np.arange(b), 1e-17)
    x = (u * sv) @ v.T
    r = _gram_chol_dd(cuda, x)
    assert np.all(np.isfinite(r))
    assert np.all(np.tril(r, -1) == 0.0)
    assert np.all(np.diag(r) >= 0.0)
    _, rh = np.linalg.qr(x)
    s_dd = np.linalg.svd(r, compute_uv=False)
    s_hh = np.linalg.svd(rh, compute_uv=False)
    np.testing.assert_allclose(s_dd, s_hh, rtol=0, atol=1e-14 * s_hh[0])
    np.testing.assert_allclose(s_dd, sv, rtol=0, atol=1e-14 * sv[0])
    # kept directions (singular values above 1e-6 of the largest): U of R^T
    kk = int(np.sum(sv > 1e-6 * sv[0]))
    ud = np.linalg.svd(r.T)[0][:, :kk]
    uh = np.linalg.svd(rh.T)[0][:, :kk]
    cos = np.linalg.svd(ud.T @ uh, compute_uv=False)
    assert np.min(cos) > 1 - 1e-12
    # columns of R^T R reproduce X^T X on the retained part
    g = x.T @ x
    np.testing.assert_allclose(r.T @ r, g, rtol=0, atol=1e-14 * np.trace(g))


def test_gram_chol_dd_zero_and_exact_rank(cuda):
    # all-zero block -> R = 0; an exactly rank-2 block -> two nonzero rows
    r = _gram_chol_dd(cuda, np.zeros((500, 8)))
    assert np.all(r == 0.0)
    rng = philox(5)
    x = rng.standard_normal((600, 2)) @ rng.standard_normal((2, 8))
    r = _gram_chol_dd(cuda, x)
    assert np.count_nonzero(np.abs(np.diag(r)) > 1e-12 * np.abs(r).max()) == 2
    np.testing.assert_allclose(r.T @ r, x.T @ x, rtol=0, atol=1e-13 * np.trace(x.T @ x))
