"""Round-2 golden vectors, made by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_r2.py

Adds (make_golden.py's files are left as they are):

* ``field_cfg3g.npz`` -- the cfg3 analogue with the noise at the full-size
  cfg3 level (std 1e-3): every one of the 40 ID pivots is gap-determined
  (SURVEY.md 8(c) gate 2), so pivots, P and the lifting are comparable
  end to end.
* ``api_cases.npz`` -- the literal API entry points on their own:
  ``accumulate_sketch(with_gram=True)`` (src/svd.py:46-68), ``power_basis``
  (src/power.py:88-112), ``finalize_svd`` single-pass (src/power.py:124-181)
  and ``build_lifting`` (src/rowid.py:115-139).

Inputs are regenerated from seeds (BLAS-free field generator or seeded
Philox draws); only the reference's OUTPUTS are stored.
"""

from __future__ import annotations

import os
import sys
import warnings
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import sketchpress as sp  # noqa: E402  (the reference, read-only)
from sketchpress.sketch import SketchOperator  # noqa: E402
from sketchpress.svd import accumulate_sketch  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

from paper_2105_01271_b200.datagen import FieldConfig, coarse_grid_indices, generate_host  # noqa: E402
import oracle  # noqa: E402  (test infrastructure: pivot gaps)

warnings.simplefilter("ignore")

# cfg3 analogue at the full-size cfg3 noise level (variance 1e-6, std 1e-3)
CFG3G = FieldConfig("cfg3g", 1000, (128, 128), 40, 0.5, 0.001, 2, 8, 100, 1, noise_std=1e-3)
API_FIELD = FieldConfig("api", 300, (32, 32), 8, 1.0, 0.005, 5, 4, 10, 1)


def grid_op(n, idx):
    spec = sp.SketchSpec(kind="injection", n=n, n_c=idx.size)
    return SketchOperator(spec=spec, idx=idx[None, :].astype(np.intp), w=np.ones((1, idx.size)))


def philox(seed):
    return np.random.Generator(np.random.Philox(seed))


def field_cfg3g(out):
    cfg = CFG3G
    a = generate_host(cfg)
    idx = coarse_grid_indices(cfg.grid, cfg.stride)
    op = grid_op(cfg.n, idx)
    kid = 40
    pc = sp.PowerConfig(q=1, columns=idx, mode="single_pass")
    fid = sp.power_id(sp.ArraySnapshotStream(a), op, kid, pc)
    orc = oracle.spc_power_id(a, idx[None, :], np.ones((1, idx.size)), idx, kid, q=1)
    runs = []
    for br, nthr in [(64, 1), (128, 1), (1000, 1), (256, os.cpu_count())]:
        with threadpool_limits(nthr):
            f2 = sp.power_id(sp.ArraySnapshotStream(a), op, kid, pc, block_rows=br)
        runs.append((sp.rel_frob_error(a, f2.reconstruct()), np.array_equal(f2.indices, fid.indices)))
    probe = philox(99).standard_normal((fid.lifting.shape[1], 2))
    rec = dict(a_checksum=np.array([a.sum(), np.abs(a).sum(), (a * a).sum()]), idx=idx,
               id_k=np.array(kid), id_p=fid.p, id_indices=fid.indices, id_skeleton=fid.skeleton,
               id_r=np.array(fid.r), id_relf=np.array(sp.rel_frob_error(a, fid.reconstruct())),
               id_gaps=orc.pivot_gaps, id_lift_probe=fid.lifting @ probe,
               id_relf_runs=np.array([r[0] for r in runs]),
               id_runs_same_pivots=np.array([r[1] for r in runs]))
    np.savez_compressed(out / "field_cfg3g.npz", **rec)
    print("cfg3g", {k: getattr(v, "shape", v) for k, v in rec.items()})


def rank_deficient(rng, m, n, rank, decay=None):
    u, _ = np.linalg.qr(rng.standard_normal((m, rank)))
    v, _ = np.linalg.qr(rng.standard_normal((n, rank)))
    s = np.linspace(2.0, 1.0, rank) if decay is None else decay
    return (u * s) @ v.T


def id_slow(out):
    """Slow spectral decay (80 values over one decade): the enriched sketch's
    spectrum spans three decades, so all 40 greedy pivots win by >= 1e-11 of
    the initial column scale and are reproducible by any FP64 implementation
    (SURVEY.md 8(c) gate 2) -- the end-to-end ID comparison (pivots, P,
    lifting) that the noise-floor fields cannot give."""
    a = rank_deficient(philox(41), 400, 2048, rank=80, decay=np.logspace(0, -1, 80))
    cols = np.arange(0, 2048, 8)
    op = grid_op(2048, cols)
    kid = 40
    pc = sp.PowerConfig(q=1, columns=cols, mode="single_pass")
    fid = sp.power_id(sp.ArraySnapshotStream(a), op, kid, pc)
    c = a[:, cols]
    gaps = oracle.pivot_gaps((c @ (c.T @ c)).T, kid)
    probe = philox(98).standard_normal((2048, 2))
    spid = sp.single_pass_id(sp.ArraySnapshotStream(a), op, 30)
    rec = dict(a=a, cols=cols, id_k=np.array(kid), id_p=fid.p, id_indices=fid.indices, id_skeleton=fid.skeleton,
               id_r=np.array(fid.r), id_relf=np.array(sp.rel_frob_error(a, fid.reconstruct())), id_gaps=gaps,
               id_lift_probe=fid.lifting @ probe, id_lift_probe_t=probe[:400].T @ fid.p,
               spid_p=spid.p, spid_indices=spid.indices, spid_r=np.array(spid.r),
               spid_lift_probe=spid.lifting @ probe,
               spid_relf=np.array(sp.rel_frob_error(a, spid.reconstruct())))
    np.savez_compressed(out / "id_slow.npz", **rec)
    print("id_slow", {k: getattr(v, "shape", v) for k, v in rec.items()})


def api_cases(out):
    rec = {}
    # 1. accumulate_sketch(with_gram=True) on a heat field with the stride-4 grid
    cfg = API_FIELD
    a = generate_host(cfg)
    idx = coarse_grid_indices(cfg.grid, cfg.stride)
    op = grid_op(cfg.n, idx)
    coarse, gram = accumulate_sketch(sp.ArraySnapshotStream(a), op, with_gram=True)
    rec.update(acc_coarse=coarse, acc_gram=gram, acc_idx=idx)
    # 2. power_basis / finalize_svd on a random full-rank problem (healthy
    #    triangular branch: every output is well conditioned)
    b = philox(31).standard_normal((60, 200))
    op1 = sp.build_sketch(sp.SketchSpec("injection", 200, 20))
    cols = np.arange(0, 200, 8)
    s0, _ = accumulate_sketch(sp.ArraySnapshotStream(b), op1)
    c = b[:, cols].copy()
    hc = b.T @ c
    basis = sp.power_basis(c, s0, sp.PowerConfig(q=1, columns=cols))
    rec.update(pb_a=b, pb_cols=cols, pb_s0=s0, pb_qb=basis.q_b, pb_rb=basis.r_b, pb_qnp=basis.q_np)
    fin = sp.finalize_svd(basis, 6, "single_pass", hc=hc, c=c, s0=s0)
    rec.update(fin_u=fin.u, fin_s=fin.s, fin_v=fin.v)
    # 3. the same with q = 2
    basis2 = sp.power_basis(c, s0, sp.PowerConfig(q=2, columns=cols))
    fin2 = sp.finalize_svd(basis2, 6, "single_pass", hc=hc, c=c, s0=s0)
    rec.update(fin2_s=fin2.s, fin2_u=fin2.u, fin2_v=fin2.v)
    # 4. build_lifting from the coarse SVD and the coarse gram
    coarse1, gram1 = accumulate_sketch(sp.ArraySnapshotStream(b), op1, with_gram=True)
    csvd = sp.thin_svd(coarse1)
    lift = sp.build_lifting(csvd, gram1, r=10, k=5)
    rec.update(bl_lift=lift, bl_coarse=coarse1, bl_gram=gram1)
    np.savez_compressed(out / "api_cases.npz", **rec)
    print("api", sorted(rec))


if __name__ == "__main__":
    with threadpool_limits(1):
        field_cfg3g(HERE)
        id_slow(HERE)
        api_cases(HERE)
