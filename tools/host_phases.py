"""Wall time of the host phases of the C2 mapping step (graph replay mode).

    python tools/host_phases.py [--steps 300]

Wraps the policy calls of optimization_step with perf_counter timers; the
sum outside `readback_wait` is the host's share of the critical path (the
next draw needs this step's loss, so steps do not pipeline).
"""

import argparse
import json
import sys
import tempfile
import time
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    args = ap.parse_args()
    import torch

    from paper_2511_23030_b200 import mapping
    from paper_2511_23030_b200.workloads import build_c2
    eng = build_c2(1_000_000, 16, store_dir=tempfile.mkdtemp())
    eng.warm_graphs()
    for s in range(20):
        eng.optimization_step(0, s)
    torch.cuda.synchronize()
    acc = defaultdict(float)

    def wrap(obj, name, label=None):
        f = getattr(obj, name)

        def w(*a, **k):
            t = time.perf_counter()
            try:
                return f(*a, **k)
            finally:
                acc[label or name] += time.perf_counter() - t
        setattr(obj, name, w)

    st = eng.store
    for n in ("ensure_resident", "mark_trained", "keyframe_get", "mark_keyframe_dirty", "segments"):
        wrap(st, n)
    for n in ("_visible_for_pose", "_finish_readback", "_precompute_next_draw", "_queue_readback"):
        wrap(eng, n)
    wrap(eng.active, "build", "active_build")
    for n in ("select_keyframe", "candidate_set", "record_loss", "overlap"):
        wrap(mapping, n)
    t0 = time.perf_counter()
    for s in range(args.steps):
        eng.optimization_step(1, s)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    out = {k: round(v / args.steps * 1e6, 1) for k, v in sorted(acc.items(), key=lambda kv: -kv[1])}
    out["_step_us"] = round(wall / args.steps * 1e6, 1)
    out["_host_outside_phases_us"] = round(out["_step_us"] - sum(v for v in out.values() if v), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
