"""Single-pass diagnostics on the GPU: the SPC-ID-ERR
streamed Gram-gap sweep against the reference's golden vectors, and the CLI
--verify pass (one streamed K8 read) against the oracle's reconstruction."""

import warnings

import numpy as np
import pytest

from conftest import load_golden, philox

import oracle
import paper_2105_01271_b200 as sp
from paper_2105_01271_b200.datagen import CONFIGS, generate_host

pytestmark = pytest.mark.gpu


def test_epsilon_sweep_matches_reference(cuda):
    g = load_golden("twopass_cases.npz")
    cfg = CONFIGS["cfg1"]
    a = generate_host(cfg)
    op, _ = sp.grid_injection(cfg.grid, cfg.stride)
    stream = sp.ArraySnapshotStream(a)
    sw = sp.streaming_epsilon_sweep(stream, op, 50)
    assert stream.passes_completed == 1 and sw.sample_stride == int(g["eps_stride"])
    np.testing.assert_allclose(sw.taus, g["eps_taus"], rtol=1e-11)
    # lambda_max of the Gram gap to ~eps (||G_f|| + tau ||G_c||): 1e-11 of the sweep's scale
    np.testing.assert_allclose(sw.values, g["eps_values"], rtol=0, atol=1e-11 * np.abs(g["eps_values"]).max())
    assert sw.min_index == int(np.argmin(g["eps_values"]))
    a2 = philox(44).standard_normal((90, 120))
    op2 = sp.build_sketch(sp.SketchSpec("injection", 120, 30))
    sw = sp.streaming_epsilon_sweep(sp.ArraySnapshotStream(a2), op2, 40)
    np.testing.assert_allclose(sw.taus, g["eps2_taus"], rtol=1e-11)
    np.testing.assert_allclose(sw.values, g["eps2_values"], rtol=0, atol=1e-11 * np.abs(g["eps2_values"]).max())
    with pytest.raises(sp.ConfigError, match="outside"):
        sp.streaming_epsilon_sweep(sp.ArraySnapshotStream(a2), op2, 0)
    with pytest.raises(sp.ConfigError, match="strictly increasing"):
        sp.streaming_epsilon_sweep(sp.ArraySnapshotStream(a2), op2, 40, taus=[2.0, 1.0])


@pytest.mark.parametrize("resident", [False, True])
def test_verify_pass_svd_and_id(cuda, resident):
    cfg = CONFIGS["cfg1"]
    a = generate_host(cfg)
    op, idx = sp.grid_injection(cfg.grid, cfg.stride)

    def stream():
        return sp.DeviceSnapshotStream(cuda.from_numpy(a).cuda()) if resident else sp.ArraySnapshotStream(a)

    s = stream()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = sp.single_pass_svd(s, op, 20)
    out = sp.verify_stream(s, res)
    assert out["extra_passes"] == 1 and s.passes_completed == 2
    np.testing.assert_allclose(out["rel_frob"], oracle.rel_frob(a, res.reconstruct()), rtol=1e-9, atol=1e-15)
    s = stream()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        fid = sp.single_pass_id(s, op, 10)
    out = sp.verify_stream(s, fid)
    np.testing.assert_allclose(out["rel_frob"], oracle.rel_frob(a, fid.reconstruct()), rtol=1e-9, atol=1e-15)
    left, right = sp.factor_pair(res)
    blocks = list(sp.reconstruct_blocks(left, right, block_rows=300))
    rec = np.vstack([b.cpu().numpy() for b in blocks])
    np.testing.assert_allclose(rec, res.reconstruct(), rtol=0, atol=1e-12 * np.abs(a).max())
