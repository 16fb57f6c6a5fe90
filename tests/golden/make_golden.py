"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

Inputs are regenerated from seeds by ``paper_2105_01271_b200.datagen`` (BLAS-free,
so the bytes are host independent) or by small seeded numpy draws recorded
here; only the reference's OUTPUTS are stored.  The files pin the oracle
(tests/test_oracle_pins.py) and give the GPU tests fixed expectations.
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
from threadpoolctl import threadpool_limits  # noqa: E402

from paper_2105_01271_b200.datagen import CONFIGS, FieldConfig, coarse_grid_indices, generate_host  # noqa: E402
import oracle  # noqa: E402  (test infrastructure: pivot gaps)

warnings.simplefilter("ignore")


def grid_op(n, idx):
    spec = sp.SketchSpec(kind="injection", n=n, n_c=idx.size)
    return SketchOperator(spec=spec, idx=idx[None, :].astype(np.intp), w=np.ones((1, idx.size)))


def philox(seed):
    return np.random.Generator(np.random.Philox(seed))


def rank_deficient(rng, m, n, rank, decay=None):
    u, _ = np.linalg.qr(rng.standard_normal((m, rank)))
    v, _ = np.linalg.qr(rng.standard_normal((n, rank)))
    s = np.linspace(2.0, 1.0, rank) if decay is None else decay
    return (u * s) @ v.T


# Small field configs (scaled analogues of cfg2/cfg3 the CPU reference finishes in seconds)
SMALL = {
    "cfg1": CONFIGS["cfg1"],
    "cfg2s": CONFIGS["cfg2"].scaled(m=400, grid=(64, 64), name="cfg2s"),
    # cfg3 analogue: 1000 x 128^2, stride 8 (n_c = 256).  Noise std scaled to
    # 1e-4 so that, as in the full-size cfg3, the kept-rank cut falls well
    # inside the signal (sigma_C boundary 2.1e-4 / 4.5e-5 vs 2.1e-4 / 5.2e-5).
    "cfg3s": FieldConfig("cfg3s", 1000, (128, 128), 40, 0.5, 0.001, 2, 8, 100, 1, noise_std=1e-4),
}


def envelope(a, op, idx, cfg, k):
    """Reference self-variability: block_rows {64,128,256,1000} x 1 thread and
    256 x all threads."""
    runs = []
    for br, nthr in [(64, 1), (128, 1), (256, 1), (1000, 1), (256, os.cpu_count())]:
        with threadpool_limits(nthr):
            if cfg.q == 0:
                res = sp.single_pass_svd(sp.ArraySnapshotStream(a), op, k, block_rows=br)
            else:
                res = sp.power_svd(sp.ArraySnapshotStream(a), op, k,
                                   sp.PowerConfig(q=cfg.q, columns=idx, mode="single_pass"), block_rows=br)
        runs.append((res.s.copy(), sp.rel_frob_error(a, res.reconstruct())))
    s = np.array([r[0] for r in runs])
    f = np.array([r[1] for r in runs])
    return s.max(0) - s.min(0), np.array(f.max() - f.min())


def field_cases(out):
    for key, cfg in SMALL.items():
        a = generate_host(cfg)
        idx = coarse_grid_indices(cfg.grid, cfg.stride)
        op = grid_op(cfg.n, idx)
        rec = {"a_checksum": np.array([a.sum(), np.abs(a).sum(), (a * a).sum()]),
               "idx": idx}
        k = min(cfg.k, idx.size - 1)
        if cfg.q == 0:
            res = sp.single_pass_svd(sp.ArraySnapshotStream(a), op, k)
        else:
            res = sp.power_svd(sp.ArraySnapshotStream(a), op, k,
                               sp.PowerConfig(q=cfg.q, columns=idx, mode="single_pass"))
        keep = 16  # leading columns only: the trailing ones are rounding noise
        rec.update(svd_u=res.u[:, :keep], svd_s=res.s, svd_v=res.v[:, :keep], svd_k=np.array(k),
                   svd_relf=np.array(sp.rel_frob_error(a, res.reconstruct())))
        env_s, env_f = envelope(a, op, idx, cfg, k)
        rec.update(svd_s_env=env_s, svd_relf_env=env_f)
        if key == "cfg3s":
            kid = 40
            fid = sp.power_id(sp.ArraySnapshotStream(a), op, kid,
                              sp.PowerConfig(q=1, columns=idx, mode="single_pass"))
            orc = oracle.spc_power_id(a, idx[None, :], np.ones((1, idx.size)), idx, kid, q=1)
            id_runs = []
            for br, nthr in [(64, 1), (128, 1), (1000, 1), (256, os.cpu_count())]:
                with threadpool_limits(nthr):
                    f2 = sp.power_id(sp.ArraySnapshotStream(a), op, kid,
                                     sp.PowerConfig(q=1, columns=idx, mode="single_pass"), block_rows=br)
                id_runs.append(sp.rel_frob_error(a, f2.reconstruct()))
            rec.update(id_relf_runs=np.array(id_runs))
            rec.update(id_k=np.array(kid), id_p=fid.p, id_indices=fid.indices,
                       id_skeleton=fid.skeleton, id_r=np.array(fid.r),
                       id_relf=np.array(sp.rel_frob_error(a, fid.reconstruct())),
                       id_gaps=orc.pivot_gaps,
                       id_lift_probe=fid.lifting @ philox(99).standard_normal(fid.lifting.shape[1]))
        np.savez_compressed(out / f"field_{key}.npz", **rec)
        print(key, {k: getattr(v, "shape", v) for k, v in rec.items()})


def small_cases(out):
    """Reference-test-style small problems (inputs regenerable from the seeds here)."""
    rec = {}
    # 1. rank-deficient power_svd with stride columns (s0 == C indices differ)
    rng = philox(6)
    a = rank_deficient(rng, 30, 80, rank=3)
    op = sp.build_sketch(sp.SketchSpec(kind="injection", n=80, n_c=16))
    r = sp.power_svd(sp.ArraySnapshotStream(a), op, 3, sp.PowerConfig(q=1, stride=5))
    rec.update(rd_s=r.s, rd_relf=np.array(sp.rel_frob_error(a, r.reconstruct())))
    # 2. full-rank random: healthy (triangular-solve) branch of single_pass_svd
    a = philox(15).standard_normal((28, 70))
    r = sp.single_pass_svd(sp.ArraySnapshotStream(a), sp.build_sketch(sp.SketchSpec("injection", 70, 10)), 5)
    rec.update(fr_s=r.s, fr_u=r.u, fr_v=r.v)
    # 3. power_svd q=2 on random full rank (healthy branch)
    a = philox(4).standard_normal((25, 50))
    r = sp.power_svd(sp.ArraySnapshotStream(a), sp.build_sketch(sp.SketchSpec("injection", 50, 10)), 4,
                     sp.PowerConfig(q=2, stride=5))
    rec.update(pq2_s=r.s, pq2_rec=r.reconstruct())
    # 4. neighbor / global stencils applied to a random block
    x = philox(21).standard_normal((5, 37))
    for kind in ("injection", "neighbor", "global"):
        o = sp.build_sketch(sp.SketchSpec(kind, 37, 9))
        rec[f"st_{kind}_idx"] = o.idx
        rec[f"st_{kind}_w"] = o.w
        rec[f"st_{kind}_out"] = sp.apply_sketch(o, x)
    # 5. pivoted QR on a graded random matrix
    m = philox(12).standard_normal((10, 8)) * np.logspace(0, -3, 8)
    f = sp.pivoted_qr(m, 6)
    rec.update(pq_perm=f.perm, pq_r=f.r, pq_q=f.q)
    # 6. row_id of a random matrix
    m = philox(1).standard_normal((9, 5))
    f = sp.row_id(m, 3)
    rec.update(rid_p=f.p, rid_idx=f.indices)
    # 7. single_pass_id exact-rank recovery problem
    a = rank_deficient(philox(10), 35, 80, rank=4)
    f = sp.single_pass_id(sp.ArraySnapshotStream(a), sp.build_sketch(sp.SketchSpec("injection", 80, 16)), 4, r=4)
    rec.update(spid_idx=f.indices, spid_p=f.p, spid_relf=np.array(sp.rel_frob_error(a, f.reconstruct())))
    # 8. gaussian-composed sketch, single_pass_svd on slow decay
    rng = philox(7)
    sv = (np.arange(60, dtype=float) + 1.0) ** -0.5
    a = rank_deficient(rng, 60, 400, rank=60, decay=sv)
    o = sp.compose_gaussian(sp.build_sketch(sp.SketchSpec("injection", 400, 40)), ell=12, seed=3)
    r = sp.single_pass_svd(sp.ArraySnapshotStream(a), o, 2)
    rec.update(gs_s=r.s, gs_relf=np.array(sp.rel_frob_error(a, r.reconstruct())), gs_omega=o.omega)
    np.savez_compressed(out / "small_cases.npz", **rec)
    print("small", sorted(rec))


def twopass_cases(out):
    """The two-pass variants: direct_svd, two_pass_svd,
    two_pass_id, power_svd / power_id in mode two_pass."""
    rec = {}
    # cfg1 field (the reference's CPU-runnable config), stride-4 grid
    cfg = CONFIGS["cfg1"]
    a = generate_host(cfg)
    idx = coarse_grid_indices(cfg.grid, cfg.stride)
    op = grid_op(cfg.n, idx)
    r = sp.two_pass_svd(sp.ArraySnapshotStream(a), op, 8)
    rec.update(tp_s=r.s, tp_u=r.u, tp_v=r.v)
    r = sp.direct_svd(sp.ArraySnapshotStream(a), op, 8, p=idx.size - 8)
    rec.update(dr_s=r.s, dr_u=r.u, dr_v=r.v)
    f = sp.two_pass_id(sp.ArraySnapshotStream(a), op, 10)
    rec.update(tpid_idx=f.indices, tpid_p=f.p, tpid_skel=f.skeleton)
    pc = sp.PowerConfig(q=1, columns=idx, mode="two_pass")
    r = sp.power_svd(sp.ArraySnapshotStream(a), op, 8, pc)
    rec.update(pwtp_s=r.s, pwtp_u=r.u, pwtp_v=r.v)
    f = sp.power_id(sp.ArraySnapshotStream(a), op, 10, pc)
    rec.update(pidtp_idx=f.indices, pidtp_p=f.p, pidtp_skel=f.skeleton)
    # random full-rank problems with 1-D injection sketches
    a = philox(33).standard_normal((60, 150))
    op1 = sp.build_sketch(sp.SketchSpec("injection", 150, 12))
    r = sp.two_pass_svd(sp.ArraySnapshotStream(a), op1, 6)
    rec.update(rtp_s=r.s, rtp_u=r.u, rtp_v=r.v)
    r = sp.direct_svd(sp.ArraySnapshotStream(a), op1, 6)
    rec.update(rdr_s=r.s, rdr_u=r.u, rdr_v=r.v)
    r = sp.power_svd(sp.ArraySnapshotStream(a), op1, 5, sp.PowerConfig(q=0, stride=6, mode="two_pass"))
    rec.update(rpw0_s=r.s, rpw0_u=r.u, rpw0_v=r.v)
    f = sp.two_pass_id(sp.ArraySnapshotStream(a), op1, 7)
    rec.update(rtpid_idx=f.indices, rtpid_p=f.p)
    # SPC-ID-ERR sweeps (src/analysis.py:141-180): cfg1 field and a random matrix
    from sketchpress.analysis import streaming_epsilon_sweep
    a = generate_host(cfg)
    sw = streaming_epsilon_sweep(sp.ArraySnapshotStream(a), op, 50)
    rec.update(eps_taus=sw.taus, eps_values=sw.values, eps_stride=np.array(sw.sample_stride))
    a2 = philox(44).standard_normal((90, 120))
    op2 = sp.build_sketch(sp.SketchSpec("injection", 120, 30))
    sw = streaming_epsilon_sweep(sp.ArraySnapshotStream(a2), op2, 40)
    rec.update(eps2_taus=sw.taus, eps2_values=sw.values, eps2_stride=np.array(sw.sample_stride))
    np.savez_compressed(out / "twopass_cases.npz", **rec)
    print("twopass", sorted(rec))


if __name__ == "__main__":
    with threadpool_limits(1):
        if len(sys.argv) > 1 and sys.argv[1] == "twopass":
            twopass_cases(HERE)
        else:
            small_cases(HERE)
            field_cases(HERE)
            twopass_cases(HERE)
