"""Device-resident C2 training in 500-step windows: host ms per step of each
window (how the per-step cost moves with the training state and the
keyframe draws over a long run).

    python tools/drift_probe.py
"""
import time, tempfile, sys, cProfile, pstats, io
sys.path.insert(0, ".")
import torch
from paper_2511_23030_b200.workloads import build_c2
eng = build_c2(1_000_000, 16, store_dir=tempfile.mkdtemp())
eng.warm_graphs()
for s in range(10): eng.optimization_step(0, s)
torch.cuda.synchronize()
for w in range(8):
    t0 = time.perf_counter()
    pr = cProfile.Profile() if w in (1, 7) else None
    if pr: pr.enable()
    for s in range(500):
        eng.optimization_step(1, w * 500 + s)
    torch.cuda.synchronize()
    if pr:
        pr.disable(); b = io.StringIO(); pstats.Stats(pr, stream=b).sort_stats("tottime").print_stats(12); print(b.getvalue()[:3000])
    dt = (time.perf_counter() - t0) / 500 * 1e3
    print("window", w, "ms/step", round(dt, 4), "spec", eng.counter_speculative, "rows", len(eng.rows), flush=True)
