"""Time of the CUDA-graph capture of a C2 mapping step (warm_graphs over the
16 keyframes with every capture timed).

    python tools/capture_probe.py
"""
import time, tempfile, sys
sys.path.insert(0, ".")
import torch
from paper_2511_23030_b200.workloads import build_c2
eng = build_c2(1_000_000, 16, store_dir=tempfile.mkdtemp())
eng.warm_graphs()
torch.cuda.synchronize()
orig = eng._capture
ts = []
def timed_capture(*a, **k):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = orig(*a, **k)
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    return r
eng._capture = timed_capture
eng.drop_graphs()
t0 = time.perf_counter()
eng.warm_graphs()
torch.cuda.synchronize()
print("warm_graphs s", round(time.perf_counter() - t0, 3), "captures", len(ts), "ms each", [round(x * 1e3, 1) for x in ts])
