#!/usr/bin/env python
"""Benchmark: single-pass power-iteration SVD (SPC-SVD + C-PWR, q = 1) on the
BASELINE cfg2 field (m = 2000 snapshots x n = 65536 = 256^2 dofs, FP64,
coarse grid stride 4 -> 4096 columns, k = 50), one GPU per rank.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config cfg2] [--no-e2e] [--no-cpu]

Metric (BASELINE.json): GB/s of A streamed.  One "step" is one complete
power_svd over the resident snapshot matrix (gather, sketch SVD, the A pass,
final factorisation); value = |A| bytes x ranks / max-over-ranks step time.
``e2e`` is the same metric through the public drop-in API from pinned host
memory (host->device copy of A and device->host copy of U, S, V inside the
timed region).  ``--impl reference`` times the CPU restatement of the
reference algorithm (oracle/, the reference is pure Python + numpy) on a
bounded sample with all host threads.

Under torchrun (N > 1) every rank factorises its own snapshot matrix
(independent datasets, weak scaling, no collective on the data path).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time
import warnings
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2105_01271_b200.datagen import CONFIGS, mode_tables  # noqa: E402

METRIC = "GB/s of A streamed (end-to-end single-pass rank-k SVD)"
UNIT = "GB/s"


# ------------------------------------------------------------------ util ----
def rank_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


_SAMPLER_SRC = r"""
import sys, time
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
print("ready", mx, flush=True)
while True:
    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
    try:
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
    except Exception:
        bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
    print(f"{time.monotonic():.6f} {sm} {bits}", flush=True)
    time.sleep(0.002)
"""


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region.

    The sampler runs in a separate process (NVML every 2 ms, timestamped) so
    it never competes with the timed loop for the interpreter lock; samples
    are kept between __enter__ and __exit__.  Falls back to nvidia-smi."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    # NVML clocks-event-reason bits (nvml.h)
    NVML_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                 "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self._proc = None
        self._mx = None
        self._t0 = self._t1 = None
        try:
            self._proc = subprocess.Popen([sys.executable, "-c", _SAMPLER_SRC, str(gpu_index)],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            line = self._proc.stdout.readline().split()
            if len(line) == 2 and line[0] == "ready":
                self._mx = line[1]
            else:
                self._proc.kill()
                self._proc = None
        except Exception:
            self._proc = None

    def __enter__(self):
        self._t0 = time.monotonic()
        return self

    def __exit__(self, *exc):
        self._t1 = time.monotonic()
        if self._proc is not None:
            time.sleep(0.005)
            self._proc.kill()
            out, _ = self._proc.communicate(timeout=10)
            for ln in out.splitlines():
                parts = ln.split()
                if len(parts) != 3:
                    continue
                t, sm, bits = float(parts[0]), parts[1], int(parts[2])
                if self._t0 <= t <= self._t1:
                    act = ["Active" if bits & self.NVML_BITS[k] else "Not Active"
                           for k in ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")]
                    self.samples.append([sm, self._mx, "", hex(bits)] + act)
        if not self.samples:
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1] and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def generate_device(cfg, torch, dev):
    """BASELINE field on the device (input setup, outside every timed region):
    A[i,(x,y)] = sum_p Sx[x,p] sum_q EC[i,(p,q)] Sy[y,q], FP64 GEMMs."""
    S, lam, coef, _ = mode_tables(cfg)
    t = np.linspace(0.0, 1.0, cfg.m)
    ec = np.exp(-np.outer(t, lam) * np.pi ** 2 * cfg.nu) * coef[None, :]
    P = cfg.modes
    EC = torch.from_numpy(ec).to(dev).view(cfg.m, P, P)
    Sx = torch.from_numpy(S[0]).to(dev)
    Sy = torch.from_numpy(S[1]).to(dev)
    T = torch.matmul(EC, Sy.t())                         # m x P(p) x gy
    A = torch.matmul(Sx, T)                              # m x gx x gy
    return A.reshape(cfg.m, cfg.n).contiguous()


def sample_config(cfg):
    """Bounded CPU sample of the workload: the first 1/8 of the grid rows
    (an x-slab of the same field), same m, same stride, same k and q."""
    gx, gy = cfg.grid
    return cfg.scaled(grid=(max(cfg.stride * 4, gx // 8), gy), name=cfg.name + "-xslab")


def time_cpu_reference(cfg, steps, warmup, threads):
    """Oracle (numpy restatement of the reference) on the bounded sample."""
    import oracle
    from threadpoolctl import threadpool_limits
    from paper_2105_01271_b200.datagen import coarse_grid_indices, generate_host
    sc = sample_config(cfg)
    a = generate_host(sc)
    idx = coarse_grid_indices(sc.grid, sc.stride)
    w = np.ones((1, idx.size))
    k = min(sc.k, idx.size - 1)
    times = []
    with threadpool_limits(threads), warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            if sc.q == 0:
                oracle.spc_svd(a, idx[None, :], w, k)
            else:
                oracle.spc_power_svd(a, idx[None, :], w, idx, k, q=sc.q)
            dt = time.perf_counter() - t0
            if i >= warmup:
                times.append(dt)
    sec = statistics.mean(times)
    return {"value": a.nbytes / sec / 1e9, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sc.m}x{sc.n} x-slab ({sc.grid[0]}x{sc.grid[1]} grid) of {cfg.name}, "
                      f"n_c={idx.size}, k={k}, q={sc.q}; oracle/ numpy restatement, "
                      f"{threads} BLAS thread(s), mean of {steps} after {warmup} warm-up",
            "sec_per_step": sec}


# ------------------------------------------------------------ our arm ----
def run_ours(args):
    import torch
    import torch.distributed as dist
    rank, world, local = rank_env()
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2105_01271_b200 as sp
    from paper_2105_01271_b200 import _lib
    from paper_2105_01271_b200.datagen import coarse_grid_indices
    from paper_2105_01271_b200.datagen import generate_device as gen_dev
    from paper_2105_01271_b200.sharded import DeviceOps, TorchComm, sharded_power_svd
    cfg = CONFIGS[args.config]
    k = cfg.k
    if world == 1:
        A = gen_dev(cfg, dev)
        op, cols = sp.grid_injection(cfg.grid, cfg.stride)
        pc = sp.PowerConfig(q=cfg.q, columns=cols)
    else:
        # weak scaling of the column-sharded algorithm: rank i owns the x-slab
        # [i*gx, (i+1)*gx) of a (world*gx) x gy grid -- the cfg2 slab per GPU
        gx = cfg.grid[0]
        gcfg = cfg.scaled(grid=(gx * world,) + tuple(cfg.grid[1:]), name=f"{cfg.name}-x{world}")
        A = gen_dev(gcfg, dev, x_range=(rank * gx, (rank + 1) * gx))
        cols = coarse_grid_indices(gcfg.grid, gcfg.stride)
        comm, dops = TorchComm(), DeviceOps()
    n_local = A.shape[1]
    a_bytes = A.numel() * A.element_size()

    class _Res:
        def __init__(self, u, r):
            self.u, self.kept_rank = u, r

    def step():
        if world > 1:
            u, s_, v, r_, _ = sharded_power_svd(A, rank * n_local, cols, k, cfg.q, comm, dops)
            return _Res(u, r_)
        stream = sp.DeviceSnapshotStream(A)
        if cfg.q == 0:
            return sp.single_pass_svd(stream, op, k, return_device=True)
        return sp.power_svd(stream, op, k, pc, return_device=True)

    def barrier():
        if world > 1:
            dist.barrier()

    warnings.simplefilter("ignore")
    # like timeit: no cyclic-GC pass (tens of ms on an interpreter holding torch)
    # inside the timed loop; collected once here, re-enabled after
    gc.collect()
    gc.disable()
    # W warm-up steps, continued until ~0.3 s of work has run so the clocks
    # and the allocator pools are at steady state when the timed loop starts
    t_w = time.perf_counter()
    done = 0
    while done < args.warmup or time.perf_counter() - t_w < 0.3:
        res = step()
        done += 1
        if done % 8 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    warm_done = done
    # ---- timed region (device events, max over ranks)
    l0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(args.steps):
            res = step()
        ev1.record()
        torch.cuda.synchronize()
        barrier()
    gc.enable()
    launches = (_lib.launch_count() - l0) // max(1, args.steps)
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = a_bytes * world / (ms * 1e-3) / 1e9

    # ---- dominant kernel: the A pass (K2) on the launching stream
    r = int(res.kept_rank)
    Z = res.u[:, :max(r, 1)].contiguous()
    Y = torch.empty((n_local, max(r, 1)), dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream()

    def apass():
        _lib.call("sp_skinny_atz", A.data_ptr(), _lib.SP_F64, cfg.m, n_local, n_local, Z.data_ptr(), Z.shape[1],
                  Z.shape[1], Y.data_ptr(), Z.shape[1], s.cuda_stream)
    for _ in range(3):
        apass()
    # A (1.05 GB at cfg2) is 8x the 126 MB L2 and K2 streams it in the same
    # order every launch, so nothing of it survives in L2 between launches:
    # no flush (a write flush would leave 256 MB of dirty lines for the next
    # launch to write back, charging K2 for traffic that is not its own)
    durs = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        apass()
        e1.record(s)
        torch.cuda.synchronize()
        durs.append(e0.elapsed_time(e1))
    apass_ms = statistics.median(durs)
    algo_bytes = a_bytes + cfg.m * Z.shape[1] * 8 + n_local * Z.shape[1] * 8
    achieved = algo_bytes / (apass_ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    traffic = None
    tp = ROOT / "profiles" / "apass_traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- e2e through the public API from pinned host memory
    e2e = None
    if not args.no_e2e:
        host = torch.empty((cfg.m, n_local), dtype=torch.float64, pin_memory=True)
        host.copy_(A)
        hv = host.numpy()
        torch.cuda.synchronize()

        class _Out:
            def __init__(self, u, s_, v):
                self.u, self.s, self.v = u, s_, v

        def e2e_step():
            if world > 1:
                # H2D of this rank's slab, the sharded pipeline, D2H of U, S, V_i
                from paper_2105_01271_b200.device import to_host_many
                ad = torch.empty((cfg.m, n_local), dtype=torch.float64, device=dev)
                ad.copy_(host, non_blocking=True)
                u, s_, v, _, _ = sharded_power_svd(ad, rank * n_local, cols, k, cfg.q, comm, dops)
                hu, hvv = to_host_many(u, v)
                return _Out(hu, s_, hvv)
            stream = sp.ArraySnapshotStream(hv)
            if cfg.q == 0:
                out = sp.single_pass_svd(stream, op, k)
            else:
                out = sp.power_svd(stream, op, k, pc)
            return out
        # warm-up: two live result sets, so the pinned staging buffers of the
        # D2H copies are in torch's host caching allocator (steady state)
        out = e2e_step()
        out = e2e_step()
        d2h = out.u.nbytes + out.s.nbytes + out.v.nbytes
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gc.collect()
        gc.disable()
        e0.record()
        n_e2e = max(1, min(args.steps, 5))
        for _ in range(n_e2e):
            out = e2e_step()
        e1.record()
        torch.cuda.synchronize()
        gc.enable()
        e_ms = e0.elapsed_time(e1) / n_e2e
        if world > 1:
            t = torch.tensor([e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": a_bytes * world / (e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": a_bytes,
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = time_cpu_reference(cfg, steps=1, warmup=1, threads=1)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE cfg2 heat field, seed 1)",
            "config": {"workload": f"{cfg.name}: power_svd single-pass q={cfg.q}, k={k}, m={cfg.m}, "
                                   f"n={cfg.n} ({cfg.grid[0]}x{cfg.grid[1]}), stride {cfg.stride} "
                                   f"-> n_c={cols.size}",
                       "a_bytes": a_bytes, "l2": "A (1.05 GB) > L2 (126 MB): inputs larger than L2",
                       "warmup_steps_run": warm_done,
                       "kept_rank": r,
                       "parallelism": ("1 GPU" if world == 1 else
                                       f"column-sharded over {world} GPUs (NCCL all-gather of C and the "
                                       f"r x r TSQR factors), one {cfg.grid[0]}x{cfg.grid[1]} x-slab per GPU "
                                       f"(weak): global grid {cfg.grid[0] * world}x{cfg.grid[1]}")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": "skinny_tma_kernel (K2, Y = A^T U_r, TMA bulk-copy pass)",
                         "launch_ms": apass_ms,
                         "algorithmic_bytes_per_launch": algo_bytes},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_reference(args):
    rank, world, _ = rank_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    threads = len(os.sched_getaffinity(0))
    res = time_cpu_reference(cfg, steps=args.steps, warmup=min(args.warmup, 1), threads=threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["sec_per_step"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE cfg2 heat field, seed 1), bounded x-slab sample",
        "config": {"workload": f"{cfg.name} sample: {res['sample']}"},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
