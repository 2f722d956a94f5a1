"""End-to-end vs device-resident steps on the same training trajectory:
windows of 4 x 50 C2 steps alternating the keyframe upload off / on, host
ms per step and eager steps of each.

    python tools/e2e_probe.py
"""
import time, tempfile, sys
sys.path.insert(0, ".")
import torch
from paper_2511_23030_b200.workloads import build_c2
eng = build_c2(1_000_000, 16, store_dir=tempfile.mkdtemp())
eng.warm_graphs()
for s in range(10): eng.optimization_step(0, s)
step = 10
for w in range(20):
    out = []
    for mode in (False, True, False, True):
        eng.upload_keyframes_each_step = mode
        torch.cuda.synchronize(); t0 = time.perf_counter()
        e0 = eng.counter_eager
        for s in range(50):
            eng.optimization_step(1, step); step += 1
        torch.cuda.synchronize()
        out.append((mode, round((time.perf_counter() - t0) / 50 * 1e3, 3), eng.counter_eager - e0))
    print("window", w, out, flush=True)
