for c in cfg3 cfg5; do timeout 900 python scripts/id_call.py $c 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_api.py tests/test_gpu_sharded.py -q -s -m gpu -p no:cacheprovider -k "id or sharded" > gpurun_out/r2_run17.log 2>&1; echo "tests rc=$?"; grep -E "cfg3 power_id|passed|failed" gpurun_out/r2_run17.log | tail -5
python - <<'PY'
import sys, time, warnings, torch
sys.path.insert(0, '.')
import paper_2105_01271_b200 as sp
from paper_2105_01271_b200.datagen import CONFIGS, generate_device
warnings.simplefilter("ignore")
for c in ("cfg3", "cfg5"):
    cfg = CONFIGS[c]; A = generate_device(cfg); op, cols = sp.grid_injection(cfg.grid, cfg.stride)
    pc = sp.PowerConfig(q=1, columns=cols)
    f = sp.power_id(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True); del f
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
    for _ in range(2): f = sp.power_id(sp.DeviceSnapshotStream(A), op, cfg.k, pc, return_device=True)
    e1.record(); torch.cuda.synchronize(); print(c, "power_id ms", e0.elapsed_time(e1) / 2, "bulk", f.lifting.bulk_split)
    del A, f; torch.cuda.empty_cache()
PY
