import sys, torch
sys.path.insert(0, '.')
from paper_2105_01271_b200 import _lib
dev = torch.device('cuda', 0); st = torch.cuda.current_stream(); s = st.cuda_stream
for rows in (4096, 16384, 262144):
    X = torch.randn(rows, 32, dtype=torch.float64, device=dev)
    R = torch.empty(32, 32, dtype=torch.float64, device=dev)
    f = lambda: _lib.call("sp_gram_chol_dd", rows, 32, X.data_ptr(), 32, R.data_ptr(), 32, s)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(20): f()
    e1.record(st); torch.cuda.synchronize()
    print(rows, e0.elapsed_time(e1) / 20 * 1e3, 'us', flush=True)
