"""Pin the CPU oracle (oracle/, test infrastructure) to the REFERENCE's own
outputs (tests/golden, produced by running /root/reference) and to the
reference test-suite's known answers.  CPU only."""

import warnings

import numpy as np
import pytest
from threadpoolctl import threadpool_limits

from conftest import load_golden, philox, rank_deficient

import oracle
from paper_2105_01271_b200.datagen import CONFIGS, FieldConfig, generate_host

SMALL = {
    "cfg1": CONFIGS["cfg1"],
    "cfg2s": CONFIGS["cfg2"].scaled(m=400, grid=(64, 64), name="cfg2s"),
    "cfg3s": FieldConfig("cfg3s", 1000, (128, 128), 40, 0.5, 0.001, 2, 8, 100, 1, noise_std=1e-4),
}


@pytest.fixture(autouse=True)
def one_thread():
    # the golden vectors were produced with one BLAS thread (block-serial,
    # bitwise reproducible at fixed block size and thread count)
    with threadpool_limits(1), warnings.catch_warnings():
        warnings.simplefilter("ignore")
        yield


def _ones(idx):
    return np.ones((1, idx.size))


@pytest.mark.parametrize("key", ["cfg1", "cfg2s", "cfg3s"])
def test_generator_bytes_and_grid(key):
    cfg = SMALL[key]
    g = load_golden(f"field_{key}.npz")
    a = generate_host(cfg)
    np.testing.assert_array_equal(np.array([a.sum(), np.abs(a).sum(), (a * a).sum()]), g["a_checksum"])
    assert np.array_equal(oracle.grid_coarse_indices(cfg.grid, cfg.stride), g["idx"])


@pytest.mark.parametrize("key", ["cfg1", "cfg2s", "cfg3s"])
def test_oracle_svd_matches_reference(key):
    cfg = SMALL[key]
    g = load_golden(f"field_{key}.npz")
    a = generate_host(cfg)
    idx = g["idx"]
    k = int(g["svd_k"])
    if cfg.q == 0:
        res = oracle.spc_svd(a, idx[None, :], _ones(idx), k)
    else:
        res = oracle.spc_power_svd(a, idx[None, :], _ones(idx), idx, k, q=cfg.q)
    # same host, same thread count, same block order: identical to the reference
    np.testing.assert_allclose(res.s, g["svd_s"], rtol=1e-13, atol=1e-15 * g["svd_s"][0])
    np.testing.assert_allclose(oracle.rel_frob(a, res.reconstruct()), float(g["svd_relf"]), rtol=1e-8)
    assert res.used_pinv


def test_oracle_power_id_matches_reference():
    cfg = SMALL["cfg3s"]
    g = load_golden("field_cfg3s.npz")
    a = generate_host(cfg)
    idx = g["idx"]
    kid = int(g["id_k"])
    res = oracle.spc_power_id(a, idx[None, :], _ones(idx), idx, kid, q=1)
    assert np.array_equal(res.indices, g["id_indices"])
    np.testing.assert_allclose(res.p, g["id_p"], atol=1e-9)
    assert res.r == int(g["id_r"])
    np.testing.assert_allclose(oracle.rel_frob(a, res.reconstruct()), float(g["id_relf"]), rtol=1e-8)
    probe = res.lifting @ philox(99).standard_normal(res.lifting.shape[1])
    np.testing.assert_allclose(probe, g["id_lift_probe"], rtol=1e-8, atol=1e-8 * np.abs(probe).max())
    np.testing.assert_allclose(res.pivot_gaps, g["id_gaps"], rtol=1e-6, atol=1e-17)


def test_oracle_small_cases_match_reference():
    g = load_golden("small_cases.npz")
    a = rank_deficient(philox(6), 30, 80, rank=3)
    idx, w = oracle.stencil_tables("injection", 80, 16)
    r = oracle.spc_power_svd(a, idx, w, np.arange(0, 80, 5), 3, q=1)
    np.testing.assert_allclose(r.s, g["rd_s"], rtol=1e-12)
    a = philox(15).standard_normal((28, 70))
    idx, w = oracle.stencil_tables("injection", 70, 10)
    r = oracle.spc_svd(a, idx, w, 5)
    np.testing.assert_allclose(r.s, g["fr_s"], rtol=1e-13)
    np.testing.assert_allclose(r.u, g["fr_u"], atol=1e-12)
    assert not r.used_pinv
    a = philox(4).standard_normal((25, 50))
    idx, w = oracle.stencil_tables("injection", 50, 10)
    r = oracle.spc_power_svd(a, idx, w, np.arange(0, 50, 5), 4, q=2)
    np.testing.assert_allclose(r.s, g["pq2_s"], rtol=1e-12)
    np.testing.assert_allclose(r.reconstruct(), g["pq2_rec"], atol=1e-12)
    x = philox(21).standard_normal((5, 37))
    for kind in ("injection", "neighbor", "global"):
        idx, w = oracle.stencil_tables(kind, 37, 9)
        assert np.array_equal(idx, g[f"st_{kind}_idx"])
        assert np.array_equal(w, g[f"st_{kind}_w"])
        assert np.array_equal(oracle.sketch_rows(x, idx, w), g[f"st_{kind}_out"])
    m = philox(12).standard_normal((10, 8)) * np.logspace(0, -3, 8)
    q, rr, perm = oracle.greedy_pivoted_qr(m, 6)
    assert np.array_equal(perm, g["pq_perm"])
    np.testing.assert_allclose(rr, g["pq_r"], atol=1e-14)
    np.testing.assert_allclose(q, g["pq_q"], atol=1e-14)
    f = oracle.interp_rows(philox(1).standard_normal((9, 5)), 3)
    assert np.array_equal(f.indices, g["rid_idx"])
    np.testing.assert_allclose(f.p, g["rid_p"], atol=1e-13)
    a = rank_deficient(philox(10), 35, 80, rank=4)
    idx, w = oracle.stencil_tables("injection", 80, 16)
    f = oracle.spc_id(a, idx, w, 4, r=4)
    assert np.array_equal(f.indices, g["spid_idx"])
    np.testing.assert_allclose(f.p, g["spid_p"], atol=1e-10)


# ---- the reference test-suite's known answers (pkg/tests), on the oracle ----
def test_hand_examples():
    idx, w = oracle.stencil_tables("injection", 4, 2)
    assert np.array_equal(oracle.sketch_rows(np.array([[1.0, 2.0, 3.0, 4.0]]), idx, w), [[1.0, 3.0]])
    idx, w = oracle.stencil_tables("neighbor", 6, 2, d=1, weights=(0.25, 0.5, 0.25))
    got = oracle.sketch_rows(np.array([[0.0, 1.0, 0.0, 0.0, 0.0, 0.0]]), idx, w)
    np.testing.assert_allclose(got[0, 0], 1.0 / 3.0)
    f = oracle.interp_rows(np.array([[1.0, 2.0], [2.0, 4.0]]), 1)
    np.testing.assert_array_equal(f.indices, [1])
    np.testing.assert_allclose(f.p, [[0.5], [1.0]])
    base = philox(10).standard_normal(4)
    m = np.column_stack([base, base, 2.0 * base, base])
    _, _, perm = oracle.greedy_pivoted_qr(m, 2)
    assert perm[0] == 2 and perm[1] == 0
    np.testing.assert_allclose(oracle.reciprocal_cut(np.array([2.0, 1.0, 0.0])), [0.5, 1.0, 0.0])
    np.testing.assert_allclose(oracle.reciprocal_cut(np.array([1.0, 1e-18])), [1.0, 0.0])
    with pytest.raises(oracle.OracleConfigError):
        oracle.reciprocal_cut(np.array([1.0, 2.0]))


def test_exact_rank_recovery():
    a = rank_deficient(philox(6), 30, 80, rank=3)
    idx, w = oracle.stencil_tables("injection", 80, 16)
    out = oracle.spc_power_svd(a, idx, w, np.arange(0, 80, 5), 3, q=1)
    assert oracle.rel_frob(a, out.reconstruct()) <= 1e-8
    fid = oracle.spc_power_id(a, idx, w, np.arange(0, 80, 5), 3, q=1)
    assert oracle.rel_frob(a, fid.reconstruct()) <= 1e-8


def test_projector_target_equals_reference_in_exact_rank_case():
    # for an exactly low-rank A both the reference and the target are exact
    a = rank_deficient(philox(3), 40, 200, rank=5)
    idx = np.arange(0, 200, 8)
    u, s, v, r = oracle.projector_target_svd(a, a[:, idx], 5, 1)
    assert r == 5
    assert oracle.rel_frob(a, (u * s) @ v.T) <= 1e-12


def _same_up_to_sign(x, y, atol):
    """Columns equal up to a per-column sign flip."""
    sgn = np.sign(np.sum(x * y, axis=0))
    sgn[sgn == 0] = 1.0
    np.testing.assert_allclose(x * sgn, y, rtol=0, atol=atol)


def test_oracle_two_pass_variants_match_reference():
    """direct_svd, two_pass_svd, two_pass_id and the
    two-pass power modes, oracle vs the reference's own outputs."""
    g = load_golden("twopass_cases.npz")
    cfg = CONFIGS["cfg1"]
    a = generate_host(cfg)
    idx = oracle.grid_coarse_indices(cfg.grid, cfg.stride)
    tab, w = idx[None, :], _ones(idx)
    r = oracle.two_pass_svd(a, tab, w, 8)
    np.testing.assert_allclose(r.s, g["tp_s"], rtol=1e-13)
    _same_up_to_sign(r.u, g["tp_u"], 1e-10)
    _same_up_to_sign(r.v, g["tp_v"], 1e-10)
    r = oracle.direct_svd(a, tab, w, 8, p=idx.size - 8)
    np.testing.assert_allclose(r.s, g["dr_s"], rtol=1e-13)
    _same_up_to_sign(r.u, g["dr_u"], 1e-10)
    _same_up_to_sign(r.v, g["dr_v"], 1e-10 * np.abs(g["dr_v"]).max())
    f = oracle.two_pass_id(a, tab, w, 10)
    assert np.array_equal(f.indices, g["tpid_idx"])
    np.testing.assert_allclose(f.p, g["tpid_p"], rtol=0, atol=1e-10)
    assert np.array_equal(f.skeleton, g["tpid_skel"])  # fine rows: exact copies
    r = oracle.power_svd_two_pass(a, tab, w, idx, 8, q=1)
    np.testing.assert_allclose(r.s, g["pwtp_s"], rtol=1e-12)
    _same_up_to_sign(r.u, g["pwtp_u"], 1e-8)
    f = oracle.power_id_two_pass(a, tab, w, idx, 10, q=1)
    assert np.array_equal(f.indices, g["pidtp_idx"])
    assert np.array_equal(f.skeleton, g["pidtp_skel"])
    # random full-rank problems, 1-D injection sketch (n=150, n_c=12)
    a = philox(33).standard_normal((60, 150))
    t1 = oracle.stencil_tables("injection", 150, 12)
    tab1, w1 = t1[0], t1[1]
    r = oracle.two_pass_svd(a, tab1, w1, 6)
    np.testing.assert_allclose(r.s, g["rtp_s"], rtol=1e-13)
    _same_up_to_sign(r.u, g["rtp_u"], 1e-11)
    r = oracle.direct_svd(a, tab1, w1, 6)
    np.testing.assert_allclose(r.s, g["rdr_s"], rtol=1e-13)
    _same_up_to_sign(r.v, g["rdr_v"], 1e-11 * np.abs(g["rdr_v"]).max())
    cols = np.arange(0, 150, 6)
    r = oracle.power_svd_two_pass(a, tab1, w1, cols, 5, q=0)
    np.testing.assert_allclose(r.s, g["rpw0_s"], rtol=1e-13)
    _same_up_to_sign(r.v, g["rpw0_v"], 1e-11)
    f = oracle.two_pass_id(a, tab1, w1, 7)
    assert np.array_equal(f.indices, g["rtpid_idx"])
    np.testing.assert_allclose(f.p, g["rtpid_p"], rtol=0, atol=1e-11)


def test_oracle_epsilon_sweep_matches_reference():
    """SPC-ID-ERR (src/analysis.py:141-180), oracle vs the reference's outputs."""
    g = load_golden("twopass_cases.npz")
    cfg = CONFIGS["cfg1"]
    a = generate_host(cfg)
    idx = oracle.grid_coarse_indices(cfg.grid, cfg.stride)
    taus, vals, stride = oracle.epsilon_sweep(a, idx[None, :], _ones(idx), 50)
    assert stride == int(g["eps_stride"])
    np.testing.assert_allclose(taus, g["eps_taus"], rtol=1e-13)
    np.testing.assert_allclose(vals, g["eps_values"], rtol=0, atol=1e-12 * np.abs(g["eps_values"]).max())
    a2 = philox(44).standard_normal((90, 120))
    t1 = oracle.stencil_tables("injection", 120, 30)
    taus, vals, stride = oracle.epsilon_sweep(a2, t1[0], t1[1], 40)
    assert stride == int(g["eps2_stride"])
    np.testing.assert_allclose(taus, g["eps2_taus"], rtol=1e-13)
    np.testing.assert_allclose(vals, g["eps2_values"], rtol=0, atol=1e-12 * np.abs(g["eps2_values"]).max())
