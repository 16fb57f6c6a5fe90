"""CPU tests: the C-ABI library loads and exports every declared symbol (no
compute without a GPU), and the host-side logic of the drop-in mirror
(streams and pass accounting, sketch tables, validation, generators)."""

import ctypes
import re
import struct
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, philox

import oracle
import paper_2105_01271_b200 as sp
from paper_2105_01271_b200 import _lib
from paper_2105_01271_b200.datagen import CONFIGS, FieldConfig, analytic_singular_values, generate_host

HEADER = ROOT / "include" / "sketchpress_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    names = declared_symbols()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)
    assert lib.sp_abi_version() == 1


def test_library_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_mapping():
    lib = _lib.load()
    with pytest.raises(sp.ConfigError):
        _lib.check(_lib.SP_ECONFIG)
    with pytest.raises(sp.NumericalError):
        _lib.check(_lib.SP_ENUMERICAL)
    with pytest.raises(sp.FormatError):
        _lib.check(_lib.SP_EIO)
    assert issubclass(sp.ConfigError, ValueError)
    assert issubclass(sp.RankDeficiencyWarning, RuntimeWarning)
    assert lib.sp_launch_count() >= 0


def test_validation_paths_need_no_gpu():
    # argument validation happens before any device work (reference order)
    with pytest.raises(sp.ConfigError):
        sp.PowerConfig(q=1, reorth=True, mode="single_pass")
    with pytest.raises(sp.ConfigError):
        sp.PowerConfig(q=-1)
    with pytest.raises(sp.ConfigError):
        sp.SketchSpec(kind="injection", n=4, n_c=5)
    with pytest.raises(sp.ConfigError):
        sp.SketchSpec(kind="neighbor", n=10, n_c=2, d=1, weights=(0.5, 0.6, 0.2))
    with pytest.raises(sp.ConfigError):
        sp.SketchSpec(kind="mystery", n=10, n_c=2)
    a = philox(1).standard_normal((10, 30))
    op = sp.build_sketch(sp.SketchSpec("injection", 30, 5))
    with pytest.raises(sp.ConfigError, match="n_c"):
        sp.single_pass_svd(sp.ArraySnapshotStream(a), op, 6)
    with pytest.raises(sp.ConfigError, match="exceed target rank"):
        sp.power_svd(sp.ArraySnapshotStream(a), op, 5, sp.PowerConfig(q=1, columns=np.arange(5)))
    with pytest.raises(sp.ConfigError, match="q >= 1"):
        sp.power_svd(sp.ArraySnapshotStream(a), op, 2, sp.PowerConfig(q=0, stride=5))
    with pytest.raises(sp.ConfigError, match="ID pipeline"):
        sp.power_id(sp.ArraySnapshotStream(a), op, 2, sp.PowerConfig(q=1, mode="two_pass", reorth=True))


# ------------------------------------------------------------- streams ----
def test_stream_pass_accounting():
    a = philox(2).standard_normal((10, 4))
    s = sp.ArraySnapshotStream(a)
    blocks = list(s.blocks(3))
    assert [b.shape[0] for b in blocks] == [3, 3, 3, 1]
    assert s.passes_completed == 1 and s.at_end_of_pass
    assert not blocks[0].flags.writeable
    s.rewind()
    s.next_block(4)
    with pytest.raises(sp.PassAuditError):
        s.rewind()
    with pytest.raises(sp.ConfigError):
        s.next_block(0)


def test_lrsm_roundtrip_and_errors(tmp_path):
    a = philox(3).standard_normal((7, 5))
    p = tmp_path / "x.lrsm"
    sp.write_snapshots(p, a)
    with sp.open_stream(p) as s:
        np.testing.assert_array_equal(sp.read_matrix(s), a)
        assert s.passes_completed == 1
    p32 = tmp_path / "y.lrsm"
    sp.write_snapshots(p32, a.astype(np.float32), scalar_kind=1)
    with sp.open_stream(p32) as s:
        blk = s.next_block(10)
        assert blk.dtype == np.float64
        np.testing.assert_array_equal(blk, a.astype(np.float32).astype(np.float64))
    raw = p.read_bytes()
    bad = tmp_path / "bad.lrsm"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(sp.FormatError, match="magic"):
        sp.open_stream(bad)
    bad.write_bytes(raw[:-8])
    with pytest.raises(sp.FormatError, match="truncated"):
        sp.open_stream(bad)
    bad.write_bytes(raw + b"\0")
    with pytest.raises(sp.FormatError, match="trailing"):
        sp.open_stream(bad)
    assert struct.unpack("<4sHBBQQ", raw[:24])[4:] == (7, 5)


def test_stream_poisoning(tmp_path):
    p = tmp_path / "z.lrsm"
    sp.write_snapshots(p, philox(4).standard_normal((6, 3)))
    s = sp.open_stream(p)
    s.next_block(2)
    s._fh.close()
    with pytest.raises(sp.StreamPoisonedError):
        s.next_block(2)
    with pytest.raises(sp.StreamPoisonedError):
        s.next_block(2)


# ------------------------------------------------------------- sketches ----
@pytest.mark.parametrize("kind", ["injection", "neighbor", "global"])
def test_build_sketch_tables_match_oracle(kind):
    rng = philox(55)
    for _ in range(20):
        n = int(rng.integers(4, 200))
        n_c = int(rng.integers(1, n + 1))
        op = sp.build_sketch(sp.SketchSpec(kind, n, n_c))
        idx, w = oracle.stencil_tables(kind, n, n_c)
        assert np.array_equal(op.idx, idx) and np.array_equal(op.w, w)
        dense = sp.explicit_matrix(op)
        x = rng.standard_normal((3, n))
        assert np.abs(oracle.sketch_rows(x, idx, w) - x @ dense).max() <= 1e-12 * np.abs(x).max()


@pytest.mark.parametrize("shape,stride", [((64, 64), 4), ((256, 256), 4), ((512, 512), 8), ((16, 8, 12), 4)])
def test_grid_injection_matches_oracle(shape, stride):
    op, cols = sp.grid_injection(shape, stride)
    assert np.array_equal(cols, oracle.grid_coarse_indices(shape, stride))
    assert op.n == int(np.prod(shape)) and op.n_c == cols.size
    assert np.all(np.diff(cols) > 0)
    assert op.is_injection_of(cols)


def test_compose_gaussian_seed_determinism():
    base = sp.build_sketch(sp.SketchSpec("injection", 30, 10))
    one = sp.compose_gaussian(base, ell=4, seed=42)
    two = sp.compose_gaussian(base, ell=4, seed=42)
    assert one.omega.tobytes() == two.omega.tobytes() and one.out_dim == 4
    with pytest.raises(sp.ConfigError):
        sp.compose_gaussian(base, ell=10, seed=0)


# ------------------------------------------------------------ generator ----
def test_analytic_singular_values_match_dense_svd():
    cfg = CONFIGS["cfg1"]
    a = generate_host(cfg)
    s_true = analytic_singular_values(cfg)
    s = np.linalg.svd(a, compute_uv=False)
    r = int(np.sum(s_true > 1e-10 * s_true[0]))
    np.testing.assert_allclose(s[:r], s_true[:r], rtol=0, atol=1e-13 * s_true[0])
    assert r >= 8


def test_generator_shapes_and_3d():
    cfg = FieldConfig("t3", 20, (8, 6, 4), 3, 1.0, 0.003, 4, 2, 5, 1, dtype="f32")
    a = generate_host(cfg)
    assert a.shape == (20, 8 * 6 * 4) and a.dtype == np.float32
    s_true = analytic_singular_values(cfg)
    s = np.linalg.svd(a.astype(np.float64), compute_uv=False)
    np.testing.assert_allclose(s[:3], s_true[:3], rtol=1e-6)


def test_factored_lifting_host_algebra():
    left = philox(5).standard_normal((6, 3))
    right = philox(6).standard_normal((3, 20))
    lift = sp.FactoredLifting(left, right)
    dense = left @ right
    x = philox(7).standard_normal((4, 6))
    np.testing.assert_allclose(x @ lift, x @ dense)
    np.testing.assert_allclose(lift @ np.ones(20), dense @ np.ones(20))
    np.testing.assert_allclose(np.asarray(lift), dense)
    assert lift.shape == (6, 20)
    f = sp.RowIDFactors(p=np.eye(6)[:, :4], indices=np.arange(4), skeleton=philox(8).standard_normal((4, 6)),
                        lifting=lift)
    np.testing.assert_allclose(f.reconstruct(), f.p @ f.skeleton @ dense)


def test_staging_chunk_plan():
    from paper_2105_01271_b200 import snapshot_io as sio
    assert sio.chunk_rows(8 << 20, 256) == 8            # cfg4 rows: 8 per 64 MB chunk
    assert sio.chunk_rows(512 << 10, 256) == 128        # cfg2 rows
    assert sio.chunk_rows(512 << 10, 7) == 7            # never more than a stream block
    assert sio.chunk_rows(1 << 30, 256) == 1
    for rows, parts in ((10, 3), (5, 8), (1 << 20, 16)):
        sp_ = sio.split_rows(rows, parts)
        assert sp_[0][0] == 0 and sp_[-1][1] == rows
        assert all(a[1] == b[0] for a, b in zip(sp_, sp_[1:])) and len(sp_) == min(rows, parts)


def test_parallel_copy_is_exact():
    from paper_2105_01271_b200 import snapshot_io as sio
    src = np.random.default_rng(3).standard_normal((300, 5000))
    dst = np.empty_like(src)
    sio._parallel_copy(dst, src)
    assert dst.tobytes() == src.tobytes()
    d32 = np.empty((300, 5000), dtype=np.float32)
    sio._parallel_copy(d32, src)                        # dtype conversion path
    assert np.array_equal(d32, src.astype(np.float32))


def test_oracle_pivots_and_gaps_agree_with_interp_rows():
    import oracle
    x = np.random.default_rng(4).standard_normal((40, 25)) * np.logspace(0, -3, 25)
    piv, gaps = oracle.greedy_pivots_and_gaps(x.T, 10)
    assert np.array_equal(piv, oracle.interp_rows(x, 10).indices)
    assert np.array_equal(gaps, oracle.pivot_gaps(x.T, 10))


def test_host_column_generator_matches_the_field():
    from paper_2105_01271_b200.datagen import CONFIGS, generate_host, generate_host_columns
    cfg = CONFIGS["cfg2"].scaled(m=50, grid=(32, 32), name="cols")
    a = generate_host(cfg)
    cols = np.array([0, 7, 33, 500, 1023])
    np.testing.assert_allclose(generate_host_columns(cfg, 20, cols), a[:20, cols], rtol=0,
                               atol=1e-13 * np.abs(a).max())
