"""The literal API entry points and the ID outputs end to end, against golden
vectors made by running the reference itself (tests/golden/make_golden_r2.py).

* accumulate_sketch(with_gram=True)   src/svd.py:46-68
* power_basis                         src/power.py:88-112
* finalize_svd (single-pass)          src/power.py:124-181
* build_lifting                       src/rowid.py:115-139
* power_id / single_pass_id: pivots, P and the lifting (probe products) on a
  problem whose 40 pivots are all gap-determined (id_slow), and the
  noise-floor field cfg3g / cfg3s (pivots to p*, P by its residual on the
  oracle's enriched sketch for the same selection).

Tolerances are written per quantity below; the healthy problems are well
conditioned, so their outputs are compared elementwise.
"""

import warnings

import numpy as np
import pytest

from conftest import load_golden, philox

import oracle
import paper_2105_01271_b200 as sp
from paper_2105_01271_b200.datagen import FieldConfig, coarse_grid_indices, generate_host

pytestmark = pytest.mark.gpu

API_FIELD = FieldConfig("api", 300, (32, 32), 8, 1.0, 0.005, 5, 4, 10, 1)
CFG3G = FieldConfig("cfg3g", 1000, (128, 128), 40, 0.5, 0.001, 2, 8, 100, 1, noise_std=1e-3)


def _sign_match(x, y, atol):
    sgn = np.sign(np.sum(x * y, axis=0))
    sgn[sgn == 0] = 1.0
    np.testing.assert_allclose(x * sgn, y, rtol=0, atol=atol)


def _grid_op(n, idx):
    return sp.SketchOperator(spec=sp.SketchSpec(kind="injection", n=n, n_c=idx.size),
                             idx=idx[None, :].astype(np.intp), w=np.ones((1, idx.size)))


def test_accumulate_sketch_with_gram(cuda):
    g = load_golden("api_cases.npz")
    a = generate_host(API_FIELD)
    idx = coarse_grid_indices(API_FIELD.grid, API_FIELD.stride)
    assert np.array_equal(idx, g["acc_idx"])
    stream = sp.ArraySnapshotStream(a)
    coarse, gram = sp.accumulate_sketch(stream, _grid_op(a.shape[1], idx), with_gram=True)
    assert stream.passes_completed == 1
    np.testing.assert_array_equal(coarse, g["acc_coarse"])          # exact copies (K1)
    # H = A^T (A D): FP64 products in another summation order (DMMA tiles)
    scale = np.abs(g["acc_gram"]).max()
    np.testing.assert_allclose(gram, g["acc_gram"], rtol=0, atol=1e-13 * scale)
    # device-resident stream, device result
    dstream = sp.DeviceSnapshotStream(cuda.from_numpy(a).cuda())
    dc, dg = sp.accumulate_sketch(dstream, _grid_op(a.shape[1], idx), with_gram=True, return_device=True)
    np.testing.assert_array_equal(dc.cpu().numpy(), g["acc_coarse"])
    np.testing.assert_allclose(dg.cpu().numpy(), g["acc_gram"], rtol=0, atol=1e-13 * scale)


def test_power_basis_matches_reference(cuda):
    g = load_golden("api_cases.npz")
    c = g["pb_a"][:, g["pb_cols"]]
    basis = sp.power_basis(c, g["pb_s0"], sp.PowerConfig(q=1, columns=g["pb_cols"]))
    # the reference's sign convention makes Q, R unique for a full-rank input
    np.testing.assert_allclose(basis.q_b, g["pb_qb"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(basis.r_b, g["pb_rb"], rtol=0, atol=1e-10 * np.abs(g["pb_rb"]).max())
    np.testing.assert_allclose(basis.q_np, g["pb_qnp"], rtol=0, atol=1e-10)
    assert basis.q_iters == 1 and not basis.reorth_used


@pytest.mark.parametrize("q", [1, 2])
def test_finalize_svd_single_pass_matches_reference(cuda, q):
    g = load_golden("api_cases.npz")
    a, cols, s0 = g["pb_a"], g["pb_cols"], g["pb_s0"]
    c = a[:, cols].copy()
    hc = a.T @ c
    basis = sp.power_basis(c, s0, sp.PowerConfig(q=q, columns=cols))
    with warnings.catch_warnings():
        warnings.simplefilter("error", sp.RankDeficiencyWarning)   # healthy branch: no warning
        res = sp.finalize_svd(basis, 6, "single_pass", hc=hc, c=c, s0=s0)
    key = "fin" if q == 1 else "fin2"
    assert res.method == "power"
    np.testing.assert_allclose(res.s, g[f"{key}_s"], rtol=1e-10)
    _sign_match(res.u, g[f"{key}_u"], 1e-9)
    _sign_match(res.v, g[f"{key}_v"], 1e-9)
    with pytest.raises(sp.ConfigError, match="hc, c, and s0"):
        sp.finalize_svd(basis, 6, "single_pass", hc=None, c=c, s0=s0)
    with pytest.raises(sp.ConfigError, match="outside the enriched basis width"):
        sp.finalize_svd(basis, 0, "single_pass", hc=hc, c=c, s0=s0)


def test_build_lifting_matches_reference(cuda):
    g = load_golden("api_cases.npz")
    csvd = sp.thin_svd(g["bl_coarse"])
    lift = sp.build_lifting(csvd, g["bl_gram"], r=10, k=5)
    np.testing.assert_allclose(lift, g["bl_lift"], rtol=0, atol=1e-10 * np.abs(g["bl_lift"]).max())
    with pytest.raises(sp.ConfigError, match="below target rank"):
        sp.build_lifting(csvd, g["bl_gram"], r=4, k=5)


# ------------------------------------------------------------- the ID ----

def test_power_id_gap_determined_end_to_end(cuda):
    """All 40 pivots gap-determined: indices bit-exact, P and both lifting
    probes elementwise against the reference."""
    g = load_golden("id_slow.npz")
    a, cols = g["a"], g["cols"]
    assert np.all(g["id_gaps"] > 1e-11)
    op = _grid_op(a.shape[1], cols)
    stream = sp.ArraySnapshotStream(a)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        fid = sp.power_id(stream, op, 40, sp.PowerConfig(q=1, columns=cols))
    assert stream.passes_completed == 1
    np.testing.assert_array_equal(fid.indices, g["id_indices"])
    np.testing.assert_array_equal(fid.skeleton, g["id_skeleton"])
    assert fid.r == int(g["id_r"])
    # P = interpolation coefficients R1^-1 R2: conditioned by the skeleton rows
    np.testing.assert_allclose(fid.p, g["id_p"], rtol=0, atol=1e-9 * np.abs(g["id_p"]).max())
    probe = philox(98).standard_normal((a.shape[1], 2))
    lp = fid.lifting @ probe
    np.testing.assert_allclose(lp, g["id_lift_probe"], rtol=0, atol=1e-9 * np.abs(g["id_lift_probe"]).max())
    e = oracle.rel_frob(a, fid.reconstruct())
    assert abs(e - float(g["id_relf"])) <= 1e-10 * float(g["id_relf"])


def test_single_pass_id_gap_determined_end_to_end(cuda):
    g = load_golden("id_slow.npz")
    a, cols = g["a"], g["cols"]
    op = _grid_op(a.shape[1], cols)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        fid = sp.single_pass_id(sp.ArraySnapshotStream(a), op, 30)
    np.testing.assert_array_equal(fid.indices, g["spid_indices"])
    assert fid.r == int(g["spid_r"])
    np.testing.assert_allclose(fid.p, g["spid_p"], rtol=0, atol=1e-9 * np.abs(g["spid_p"]).max())
    probe = philox(98).standard_normal((a.shape[1], 2))
    np.testing.assert_allclose(fid.lifting @ probe, g["spid_lift_probe"], rtol=0,
                               atol=1e-9 * np.abs(g["spid_lift_probe"]).max())
    e = oracle.rel_frob(a, fid.reconstruct())
    assert abs(e - float(g["spid_relf"])) <= 1e-10 * float(g["spid_relf"])


def _noise_floor_id(cuda, cfg, golden):
    """Noise-floor fields: pivots past p* are rounding-decided in the reference
    too.  Gate: pivots equal up to p*; P judged by its residual on the oracle's
    enriched sketch for OUR selection (against the least-squares optimum and
    the reference's residual)."""
    g = load_golden(golden)
    a = generate_host(cfg)
    idx = coarse_grid_indices(cfg.grid, cfg.stride)
    kid = int(g["id_k"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        fid = sp.power_id(sp.ArraySnapshotStream(a), _grid_op(a.shape[1], idx), kid,
                          sp.PowerConfig(q=1, columns=idx))
    gaps = g["id_gaps"]
    below = np.flatnonzero(gaps <= 1e-13)
    pstar = int(below[0]) if below.size else kid
    same = int(np.argmax(fid.indices != g["id_indices"])) if np.any(fid.indices != g["id_indices"]) else kid
    print(f"{cfg.name}: p* = {pstar}, identical pivot prefix {same} of {kid}")
    np.testing.assert_array_equal(fid.indices[:pstar], g["id_indices"][:pstar])
    np.testing.assert_array_equal(fid.p[fid.indices], np.eye(kid))
    c = a[:, idx]
    e = c @ (c.T @ c)
    sel = fid.indices
    res_gpu = np.linalg.norm(e - fid.p @ e[sel]) / np.linalg.norm(e)
    coef, *_ = np.linalg.lstsq(e[sel].T, e.T, rcond=None)
    res_opt = np.linalg.norm(e - coef.T @ e[sel]) / np.linalg.norm(e)
    res_ref = np.linalg.norm(e - g["id_p"] @ e[g["id_indices"]]) / np.linalg.norm(e)
    print(f"{cfg.name}: ||E - P E[sel]||/||E||: ours {res_gpu:.4e}, optimum for our selection {res_opt:.4e}, "
          f"reference {res_ref:.4e}")
    # The coefficients R1^-1 R2 of a noise-floor selection are conditioned by
    # cond(E[sel]) (~1e10 here): elementwise they agree only to ~cond * eps
    # (measured 2e-5 at cfg3g with all 40 pivots identical), so P is judged by
    # what it is for -- its interpolation residual -- against the reference's
    # own P (its triangular / pinv solve) and the least-squares optimum.
    assert res_gpu <= max(res_opt * (1 + 1e-6), res_ref * (1 + 1e-2)) + 1e-16
    return fid, a, g


def test_power_id_noise_floor_cfg3g(cuda):
    fid, a, g = _noise_floor_id(cuda, CFG3G, "field_cfg3g.npz")
    assert fid.r == int(g["id_r"])
    e = oracle.rel_frob(a, fid.reconstruct())
    runs = np.append(g["id_relf_runs"], float(g["id_relf"]))
    print(f"cfg3g: ID relF ours {e:.6e}, reference runs {runs.min():.6e} .. {runs.max():.6e}")
    assert e <= runs.max() * (1 + 1e-3) + 1e-12


def test_power_id_noise_floor_cfg3s(cuda):
    cfg = FieldConfig("cfg3s", 1000, (128, 128), 40, 0.5, 0.001, 2, 8, 100, 1, noise_std=1e-4)
    _noise_floor_id(cuda, cfg, "field_cfg3s.npz")
