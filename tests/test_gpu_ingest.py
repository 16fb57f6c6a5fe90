"""Host -> HBM ingest: the page-locked staging ring
for pageable arrays and LRSM files, the direct path for page-locked arrays,
the fused per-chunk gather, and the pass accounting of src/snapshot_io.py:77-152.
Bit-exact: the staged matrix and the gathered sketch equal the source bytes."""

import numpy as np
import pytest

from conftest import philox

import paper_2105_01271_b200 as sp
from paper_2105_01271_b200 import snapshot_io as sio
from paper_2105_01271_b200.svd import _sketch_on_ingest

pytestmark = pytest.mark.gpu


def _stage(stream, block_rows, op=None, cols=None):
    s0, c, on_block = (None, None, None)
    if op is not None:
        s0, c, on_block = _sketch_on_ingest(op, stream.m, cols)
    st = sio.stage_stream(stream, block_rows, on_block)
    return st, s0, c


@pytest.mark.parametrize("block_rows", [1, 7, 256, 5000])
def test_pageable_array_through_the_ring(cuda, block_rows, monkeypatch):
    monkeypatch.setattr(sio, "CHUNK_BYTES", 1 << 20)  # many chunks, ring wrap-around
    a = philox(60).standard_normal((700, 3000))
    a[3, 5] = -0.0
    op = sp.build_sketch(sp.SketchSpec("injection", 3000, 300))
    cols = np.arange(0, 3000, 7)
    stream = sp.ArraySnapshotStream(a)
    st, s0, c = _stage(stream, block_rows, op, cols)
    assert stream.passes_completed == 1 and stream.cursor == 700
    got = st.a.cpu().numpy()
    assert got.tobytes() == a.tobytes()
    np.testing.assert_array_equal(s0.cpu().numpy(), sp.apply_sketch(op, a))
    np.testing.assert_array_equal(c.cpu().numpy(), a[:, cols])
    assert st.h2d_bytes == a.nbytes


def test_pinned_array_is_copied_directly(cuda):
    a = philox(61).standard_normal((300, 2000))
    ht = cuda.from_numpy(a).pin_memory()
    pinned = ht.numpy()
    assert sio._is_pinned(cuda, pinned)
    st, _, _ = _stage(sp.ArraySnapshotStream(pinned), 64)
    assert st.a.cpu().numpy().tobytes() == a.tobytes()


@pytest.mark.parametrize("kind", [0, 1])
def test_lrsm_file_through_the_ring(cuda, tmp_path, kind, monkeypatch):
    monkeypatch.setattr(sio, "CHUNK_BYTES", 1 << 20)
    a = philox(62).standard_normal((513, 2100))
    if kind == 1:
        a = a.astype(np.float32)
    path = tmp_path / "a.lrsm"
    sp.write_snapshots(path, a, scalar_kind=kind)
    with sp.open_stream(path) as stream:
        st, _, _ = _stage(stream, 100)
        assert stream.passes_completed == 1
        got = st.a.cpu().numpy()
        assert got.dtype == (np.float32 if kind == 1 else np.float64)
        assert got.tobytes() == a.tobytes()
        # the reference's pass audit: a second pass needs a rewind
        stream.rewind()
        st2, _, _ = _stage(stream, 1000)
        assert stream.passes_completed == 2 and st2.a.cpu().numpy().tobytes() == a.tobytes()


def test_truncated_file_poisons_the_stream(cuda, tmp_path):
    a = philox(63).standard_normal((50, 400))
    path = tmp_path / "a.lrsm"
    sp.write_snapshots(path, a)
    stream = sp.open_stream(path)
    # truncate after opening (the header check passed): the pass must fail loudly
    with open(path, "r+b") as fh:
        fh.truncate(sio.HEADER_BYTES + 20 * 400 * 8)
    with pytest.raises(sp.StreamPoisonedError):
        _stage(stream, 16)
    with pytest.raises(sp.StreamPoisonedError):
        stream.next_block(4)
    stream.close()


def test_power_svd_from_a_pageable_array_and_a_file_agree(cuda, tmp_path):
    import warnings
    from paper_2105_01271_b200.datagen import CONFIGS, generate_host
    cfg = CONFIGS["cfg2"].scaled(m=300, grid=(48, 48), name="ingest")
    a = generate_host(cfg)
    op, idx = sp.grid_injection(cfg.grid, cfg.stride)
    path = tmp_path / "f.lrsm"
    sp.write_snapshots(path, a)
    pc = sp.PowerConfig(q=1, columns=idx)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        r1 = sp.power_svd(sp.ArraySnapshotStream(a), op, 10, pc)
        with sp.open_stream(path) as fs:
            r2 = sp.power_svd(fs, op, 10, pc, block_rows=33)
            assert fs.passes_completed == 1
    assert r1.s.tobytes() == r2.s.tobytes()
    assert r1.u.tobytes() == r2.u.tobytes() and r1.v.tobytes() == r2.v.tobytes()


def test_result_buffers_are_leased_not_shared(cuda):
    """Results land in page-locked buffers leased from a pool (device.to_host_many):
    two live results never share memory, and a dropped result's buffer is
    reused by the next call."""
    import gc

    from paper_2105_01271_b200 import device as dv
    x = cuda.arange(600000, dtype=cuda.float64, device="cuda").reshape(3000, 200)   # 4.8 MB: pooled
    small = cuda.arange(10, dtype=cuda.float64, device="cuda")                      # torch's allocator
    a, s = dv.to_host_many(x, small)
    b, = dv.to_host_many(x * 2.0)
    assert not np.shares_memory(a, b)
    np.testing.assert_array_equal(a, np.arange(600000.0).reshape(3000, 200))
    np.testing.assert_array_equal(b, 2.0 * a)
    np.testing.assert_array_equal(s, np.arange(10.0))
    view = a[5:7, :3]
    addr = a.ctypes.data
    del a
    gc.collect()
    c, = dv.to_host_many(x + 1.0)           # `view` still holds a's lease: no reuse
    assert c.ctypes.data != addr
    np.testing.assert_array_equal(view, np.arange(600000.0).reshape(3000, 200)[5:7, :3])
    del view
    gc.collect()
    d, = dv.to_host_many(x + 3.0)           # a's buffer is back in the pool
    assert d.ctypes.data == addr
    np.testing.assert_array_equal(d[0, :3], [3.0, 4.0, 5.0])
    np.testing.assert_array_equal(c[0, :3], [1.0, 2.0, 3.0])


def test_release_workspaces_between_calls(cuda):
    """sp_release_workspaces hands the cached workspaces back to the driver; the
    next call re-allocates and gives the same bits."""
    from paper_2105_01271_b200 import _lib
    from paper_2105_01271_b200.datagen import CONFIGS, generate_host
    cfg = CONFIGS["cfg2"].scaled(m=300, grid=(64, 64), name="rel")
    a = generate_host(cfg)
    op, cols = sp.grid_injection(cfg.grid, cfg.stride)
    pc = sp.PowerConfig(q=1, columns=cols)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        r1 = sp.power_svd(sp.ArraySnapshotStream(a), op, 20, pc)
        free0 = cuda.cuda.mem_get_info()[0]
        _lib.release_workspaces()
        free1 = cuda.cuda.mem_get_info()[0]
        r2 = sp.power_svd(sp.ArraySnapshotStream(a), op, 20, pc)
    assert free1 >= free0
    np.testing.assert_array_equal(r1.s, r2.s)
    np.testing.assert_array_equal(r1.u, r2.u)


def test_workspace_drain_under_memory_pressure(cuda):
    """The library keeps freed workspaces of every size (csrc/workspace.cu).  When
    the device is nearly full, a call whose workspace no longer fits must drain
    those cached blocks, retry and give the same bits as without the pressure."""
    import warnings
    from paper_2105_01271_b200 import _lib
    from paper_2105_01271_b200.datagen import CONFIGS, generate_device
    cfg = CONFIGS["cfg2"].scaled(m=2000, grid=(256, 256), name="press")
    a = generate_device(cfg, cuda.device("cuda", 0))
    op, cols = sp.grid_injection(cfg.grid, 2)               # n_c = 16384: a 262 MB column block at m = 2000
    pc = sp.PowerConfig(q=1, columns=cols)
    small = a[:1500]                                        # 197 MB column block: another size class
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _lib.release_workspaces()
        want = sp.power_svd(sp.DeviceSnapshotStream(small), op, 20, pc)
        _lib.release_workspaces()
        cuda.cuda.empty_cache()
        big = sp.power_svd(sp.DeviceSnapshotStream(a), op, 20, pc)      # leaves > 262 MB in the free lists
        cuda.cuda.synchronize()
        free = cuda.cuda.mem_get_info()[0]
        keep = 128 << 20
        hog = cuda.empty(free - keep, dtype=cuda.uint8, device="cuda")  # the caller fills the device
        assert cuda.cuda.mem_get_info()[0] < 1500 * cols.size * 8      # the 197 MB block cannot be allocated
        got = sp.power_svd(sp.DeviceSnapshotStream(small), op, 20, pc)
        cuda.cuda.synchronize()
        del hog
    assert big.kept_rank >= 1
    np.testing.assert_array_equal(got.s, want.s)
    np.testing.assert_array_equal(got.u, want.u)
    np.testing.assert_array_equal(got.v, want.v)
    _lib.release_workspaces()
    cuda.cuda.empty_cache()
