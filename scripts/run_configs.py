"""Run the BASELINE configurations at full size on one GPU (evidence run).

    python scripts/run_configs.py [cfg2 cfg3 cfg4 cfg5]

For each: generate A on the device (datagen.generate_device), run the
single-pass calls the config names, time them with CUDA events, check the
kept singular values against the analytic spectrum (noise-free configs) and
report rel-Frobenius through the streamed residual kernel (K8).  Prints one
JSON line per call.
"""
import json
import sys
import time
import warnings
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp  # noqa: E402
from paper_2105_01271_b200.datagen import CONFIGS, analytic_singular_values, generate_device  # noqa: E402

warnings.simplefilter("ignore")


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / reps


def main(names):
    for name in names:
        cfg = CONFIGS[name]
        t0 = time.perf_counter()
        A = generate_device(cfg)
        torch.cuda.synchronize()
        gen_s = time.perf_counter() - t0
        op, cols = sp.grid_injection(cfg.grid, cfg.stride)
        pc = sp.PowerConfig(q=cfg.q, columns=cols)
        a_bytes = A.numel() * A.element_size()
        k = cfg.k
        res, ms = timed(lambda: sp.power_svd(sp.DeviceSnapshotStream(A), op, k, pc, return_device=True))
        r = res.kept_rank
        s = res.s.cpu().numpy()
        line = {"config": name, "call": "power_svd", "m": cfg.m, "n": cfg.n, "n_c": int(cols.size), "k": k,
                "dtype": cfg.dtype, "gen_s": round(gen_s, 1), "ms": ms, "GBps_A": a_bytes / ms / 1e6,
                "kept_rank": int(r), "s_head": s[:min(r, 8)].tolist()}
        if not cfg.noise_std:
            st = analytic_singular_values(cfg)
            line["max_abs_dsigma_over_s1_vs_analytic"] = float(np.max(np.abs(s[:r] - st[:r])) / st[0])
        rf = sp.rel_frob_error_device(A, res.u[:, :r].contiguous(), res.s[:r].contiguous(),
                                      res.v[:, :r].contiguous()) if r <= 64 else None
        line["rel_frob"] = rf
        if not cfg.noise_std:
            st = analytic_singular_values(cfg)
            line["eckart_young_rel_frob_rank_r"] = float(np.sqrt(np.sum(st[r:] ** 2) / np.sum(st ** 2)))
        print(json.dumps(line), flush=True)
        if name in ("cfg3", "cfg5"):
            fid, ms_id = timed(lambda: sp.power_id(sp.DeviceSnapshotStream(A), op, k, pc, return_device=True),
                               reps=1)
            print(json.dumps({"config": name, "call": "power_id", "k": k, "ms": ms_id, "lift_r": fid.r,
                              "first_pivots": fid.indices[:10].cpu().tolist()}), flush=True)
        del A, res
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"])
