"""GPU probe: where the end-to-end (host buffers) time goes at cfg2."""
import sys, time, warnings
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2105_01271_b200 as sp
from paper_2105_01271_b200.snapshot_io import stage_stream
from paper_2105_01271_b200.datagen import CONFIGS
from bench import generate_device
warnings.simplefilter("ignore")
cfg = CONFIGS["cfg2"]; A = generate_device(cfg, torch, torch.device("cuda", 0))
host = torch.empty(A.shape, dtype=torch.float64, pin_memory=True); host.copy_(A); hv = host.numpy()
op, cols = sp.grid_injection(cfg.grid, cfg.stride); pc = sp.PowerConfig(q=1, columns=cols)
def t(label, fn, reps=3):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): out = fn()
    torch.cuda.synchronize(); print(f"{label:40s} {(time.perf_counter()-t0)/reps*1e3:8.2f} ms"); return out
t("stage only (block_rows=256)", lambda: stage_stream(sp.ArraySnapshotStream(hv), 256))
t("stage only (block_rows=2000)", lambda: stage_stream(sp.ArraySnapshotStream(hv), 2000))
t("power_svd host stream -> device result", lambda: sp.power_svd(sp.ArraySnapshotStream(hv), op, 50, pc, return_device=True))
t("power_svd host stream -> numpy result", lambda: sp.power_svd(sp.ArraySnapshotStream(hv), op, 50, pc))
r = sp.power_svd(sp.ArraySnapshotStream(hv), op, 50, pc, return_device=True)
t("D2H of U,S,V (pageable)", lambda: (r.u.cpu(), r.s.cpu(), r.v.cpu()))
