"""Where do the device ID pivots leave the reference's at full cfg3?
Separates the enrichment E = C (C^T C) (device DMMA GEMM vs host BLAS) from
the greedy pivoted QR (device K7 vs the oracle loop)."""
import sys, json, warnings
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle
import paper_2105_01271_b200 as sp
from paper_2105_01271_b200.power import _mm
from paper_2105_01271_b200.datagen import CONFIGS, generate_device
from threadpoolctl import threadpool_limits
warnings.simplefilter("ignore")
cfg = CONFIGS["cfg3"]
A = generate_device(cfg)
op, idx = sp.grid_injection(cfg.grid, cfg.stride)
fid = sp.power_id(sp.DeviceSnapshotStream(A), op, 100, sp.PowerConfig(q=1, columns=idx), return_device=True)
piv_pipe = fid.indices.cpu().numpy()
c = A[:, torch.from_numpy(idx).cuda()].contiguous()
e_dev = _mm(0, 0, c, _mm(1, 0, c, c))
e_cublas = c @ (c.T @ c)
piv_dev = sp.row_id(e_dev, 100).indices.cpu().numpy()
piv_devcub = sp.row_id(e_cublas, 100).indices.cpu().numpy()
ch = c.cpu().numpy()
eh_dev = e_dev.cpu().numpy()
with threadpool_limits(16):
    e_np = ch @ (ch.T @ ch)
piv_np, gaps = oracle.greedy_pivots_and_gaps(e_np.T, 100)
piv_np_on_dev_e, _ = oracle.greedy_pivots_and_gaps(eh_dev.T, 100)
f = lambda x, y: int(np.argmax(x != y)) if np.any(x != y) else 100
out = {"E rel diff dev vs np": float(np.abs(eh_dev - e_np).max() / np.abs(e_np).max()),
       "E rel diff cublas vs np": float(np.abs(e_cublas.cpu().numpy() - e_np).max() / np.abs(e_np).max()),
       "pipeline vs row_id(E_dev)": f(piv_pipe, piv_dev),
       "K7(E_dev) vs oracle(E_np)": f(piv_dev, piv_np),
       "oracle(E_dev) vs oracle(E_np)": f(piv_np_on_dev_e, piv_np),
       "K7(E_dev) vs oracle(E_dev)": f(piv_dev, piv_np_on_dev_e),
       "K7(E_cublas) vs oracle(E_np)": f(piv_devcub, piv_np)}
print(json.dumps(out))
np.savez("gpurun_out/r2_pivots.npz", piv_pipe=piv_pipe, piv_dev=piv_dev, piv_np=piv_np,
         piv_np_on_dev_e=piv_np_on_dev_e, gaps=gaps)
