"""Size-general dense kernels of the drop-in (src/kernels.py:74-94): thin_qr /
thin_svd beyond the 256-column sketch cores (panel TSQR + one-sided Jacobi on
the rows of R + orthonormal completion of the null directions), and the
literal API paths that need them at full BASELINE size: two_pass_svd,
direct_svd and power_svd(mode="two_pass") on cfg2 (src/svd.py:80-143,
src/power.py:243-249) against the oracle on the same bytes.

Tolerances: sigma to 1e-12 * sigma_1 absolute (and 1e-10 relative where
sigma_i >= 1e-3 sigma_1); factors orthonormal to 1e-10; reconstructions to
1e-12 relative; the rank-deficient directions (sigma ~ 1e-16 sigma_1) are
compared only through orthonormality (they are rounding noise in LAPACK too).
"""

import warnings

import numpy as np
import pytest

from conftest import philox, rank_deficient

import oracle
import paper_2105_01271_b200 as sp
from paper_2105_01271_b200.datagen import CONFIGS, generate_host

pytestmark = pytest.mark.gpu


def _check_svd(x, fac, rank=None):
    u, s, v = fac.u, fac.s, fac.v
    p = min(x.shape)
    assert u.shape == (x.shape[0], p) and v.shape == (x.shape[1], p) and s.shape == (p,)
    st = np.linalg.svd(x, compute_uv=False)
    assert np.all(np.diff(s) <= 0) and np.all(s >= 0)
    np.testing.assert_allclose(s, st, rtol=0, atol=1e-12 * st[0])
    big = st >= 1e-3 * st[0]
    np.testing.assert_allclose(s[big], st[big], rtol=1e-10)
    np.testing.assert_allclose(u.T @ u, np.eye(p), atol=1e-10)
    np.testing.assert_allclose(v.T @ v, np.eye(p), atol=1e-10)
    np.testing.assert_allclose((u * s) @ v.T, x, rtol=0, atol=1e-12 * np.abs(x).max() * np.sqrt(p))
    # the reference's sign convention on U (src/kernels.py:52-71)
    for j in range(p):
        col = u[:, j]
        lead = np.flatnonzero(np.abs(col) > 1e-12 * np.abs(col).max())[0]
        assert col[lead] >= 0


@pytest.mark.parametrize("shape", [(600, 400), (400, 600), (1500, 1100)])
def test_thin_svd_beyond_256_full_rank(cuda, shape):
    x = philox(51).standard_normal(shape)
    _check_svd(x, sp.thin_svd(x))


@pytest.mark.parametrize("shape", [(300, 256), (256, 300), (700, 130), (64, 64), (900, 520), (33, 33)])
@pytest.mark.parametrize("decades", [9.0, 13.0])
def test_thin_svd_graded_haar_mixed_is_orthonormal(cuda, shape, decades):
    """A graded spectrum (down to 1e-13 sigma_1) mixed by Haar factors: the core has no
    grading of its own, so the normalised Jacobi columns of the small sigma_j carry a
    relative error eps sigma_1 / sigma_j (scripts/fuzz_dense.py seed 30873: 300 x 256,
    U^T U - I = 9e-4 before those columns were re-orthonormalised).  The reference's
    gesdd factors are orthonormal to eps whatever the spectrum (src/kernels.py:87-94)."""
    rng = np.random.default_rng(30873)
    rows, cols = shape
    p = min(rows, cols)
    u, _ = np.linalg.qr(rng.standard_normal((rows, p)))
    v, _ = np.linalg.qr(rng.standard_normal((cols, p)))
    x = (u * np.logspace(0, -decades, p)) @ v.T
    _check_svd(x, sp.thin_svd(x))


@pytest.mark.parametrize("shape", [(2000, 3000), (3000, 2000)])
def test_thin_svd_beyond_256_rank_deficient(cuda, shape):
    """A sketch-like matrix: numerical rank 17 (the cfg2 coarse sketch), the
    other directions completed to an orthonormal basis."""
    sv = np.logspace(0, -9, 17)
    x = rank_deficient(philox(52), shape[0], shape[1], rank=17, decay=sv)
    fac = sp.thin_svd(x)
    _check_svd(x, fac)
    assert fac.rank() == 17


@pytest.mark.parametrize("shape", [(900, 700), (700, 900), (2000, 4096)])
def test_thin_qr_beyond_256(cuda, shape):
    x = philox(53).standard_normal(shape)
    f = sp.thin_qr(x)
    p = min(shape)
    assert f.q.shape == (shape[0], p) and f.r.shape == (p, shape[1])
    np.testing.assert_allclose(f.q.T @ f.q, np.eye(p), atol=1e-11)
    np.testing.assert_allclose(f.q @ f.r, x, rtol=0, atol=1e-12 * np.abs(x).max() * np.sqrt(p))
    assert np.all(np.abs(np.tril(f.r[:, :p], -1)) <= 1e-12 * np.abs(x).max())
    # reference: numpy QR + the sign convention
    q_ref = oracle.qr_reduced(x)[0]
    np.testing.assert_allclose(f.q, q_ref, rtol=0, atol=1e-9)


def test_numerical_rank_beyond_256(cuda):
    x = rank_deficient(philox(54), 500, 700, rank=300)
    assert sp.numerical_rank(x) == 300
    assert abs(sp.spectral_norm(x) - 2.0) <= 1e-12


# --------------------------------------------- literal API at full cfg2 ----

@pytest.fixture(scope="module")
def cfg2_field():
    cfg = CONFIGS["cfg2"]
    a = generate_host(cfg)
    op, idx = sp.grid_injection(cfg.grid, cfg.stride)
    return cfg, a, op, idx


def _gate_lowrank(name, res, want, k):
    """sigma against the oracle run on the same bytes; the leading stable
    subspaces by principal angles (U / V columns are sign-ambiguous)."""
    s, ws = np.asarray(res.s), np.asarray(want.s)
    d = np.abs(s - ws)
    print(f"{name}: max |ds|/s_1 = {d.max() / ws[0]:.2e}; leading |ds_i|/s_i = "
          f"{np.array2string((d / ws)[:8], precision=1)}")
    assert np.all(d <= 1e-12 * ws[0])
    stable = ws >= 1e-3 * ws[0]
    assert np.all(d[stable] <= 1e-10 * ws[stable])
    j = int(np.count_nonzero(stable))
    assert oracle.principal_angle(np.asarray(res.u)[:, :j], want.u[:, :j]) <= 1e-8
    vr = np.asarray(res.v)[:, :j]
    vw = want.v[:, :j]
    if getattr(res, "v_orthonormal", True):
        assert oracle.principal_angle(vr, vw) <= 1e-8
    else:  # direct_svd: V = A^T U_k / s_k, column by column (sign of U's column)
        sgn = np.sign(np.sum(np.asarray(res.u)[:, :j] * want.u[:, :j], axis=0))
        err = np.linalg.norm(vr * sgn - vw, axis=0) / np.linalg.norm(vw, axis=0)
        print(f"{name}: V columns rel err {np.array2string(err, precision=1)}")
        assert np.all(err <= 1e-8)


def test_two_pass_svd_full_cfg2(cuda, cfg2_field):
    from threadpoolctl import threadpool_limits
    cfg, a, op, idx = cfg2_field
    # the coarse sketch's numerical rank is 17: the reference refuses k = 50
    with pytest.raises(sp.NumericalError, match="below target rank"):
        sp.two_pass_svd(sp.ArraySnapshotStream(a), op, cfg.k)
    k = 12
    stream = sp.ArraySnapshotStream(a)
    res = sp.two_pass_svd(stream, op, k)
    assert stream.passes_completed == 2 and res.method == "two_pass"
    w = np.ones((1, idx.size))
    with threadpool_limits(1):
        want = oracle.two_pass_svd(a, idx[None, :], w, k)
    _gate_lowrank("two_pass_svd cfg2", res, want, k)


def test_direct_svd_full_cfg2(cuda, cfg2_field):
    from threadpoolctl import threadpool_limits
    cfg, a, op, idx = cfg2_field
    k = 12   # direct_svd needs sigma_k above the 1e-12 cut (the coarse rank is 17)
    res = sp.direct_svd(sp.ArraySnapshotStream(a), op, k)
    with threadpool_limits(1):
        want = oracle.direct_svd(a, idx[None, :], np.ones((1, idx.size)), k)
    _gate_lowrank("direct_svd cfg2", res, want, k)
    with pytest.raises(sp.NumericalError, match="below target rank"):
        sp.direct_svd(sp.ArraySnapshotStream(a), op, 20)


def test_power_svd_two_pass_full_cfg2(cuda, cfg2_field):
    from threadpoolctl import threadpool_limits
    cfg, a, op, idx = cfg2_field
    stream = sp.ArraySnapshotStream(a)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = sp.power_svd(stream, op, cfg.k, sp.PowerConfig(q=1, columns=idx, mode="two_pass"))
    assert stream.passes_completed == 2
    with threadpool_limits(1):
        want = oracle.power_svd_two_pass(a, idx[None, :], np.ones((1, idx.size)), idx, cfg.k, q=1)
    _gate_lowrank("power_svd two_pass cfg2", res, want, cfg.k)


def test_single_pass_q0_rank_beyond_256_matches_oracle_kept_rank(cuda):
    """A sketch whose numerical rank exceeds the randomized block (the q = 0
    single_pass_svd of a noisy field): the device keeps every direction the
    reference keeps (exact fallback), never a truncated projector."""
    from threadpoolctl import threadpool_limits
    rng = philox(55)
    m, n = 600, 4096
    a = rank_deficient(rng, m, n, rank=320, decay=np.logspace(0, -6, 320))
    op = sp.build_sketch(sp.SketchSpec("injection", n, 400))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = sp.single_pass_svd(sp.ArraySnapshotStream(a), op, 20)
    with threadpool_limits(1):
        tu, ts, tv, r = oracle.projector_target_svd(a, a[:, op.idx[0]], 20, 1)
    assert res.kept_rank == r and r > 256
    np.testing.assert_allclose(res.s, ts[:20], rtol=1e-10, atol=1e-12 * ts[0])
