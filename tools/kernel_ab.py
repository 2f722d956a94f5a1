"""Fixed-state kernel timing for A/B of library builds.

    SM_LIB_VARIANT=<name> python tools/kernel_ab.py [--reps 20]

The C2 scene as generated (no training: every build sees exactly the same
splats), each of its 16 keyframes rendered forward + loss + backward `reps`
times (gradients accumulate, no Adam, so nothing changes between builds or
repetitions).  Prints one JSON line: the per-stage times from the in-graph
CUDA events and the whole pass timed without them.  bench.py trains while it
measures, so two builds that round differently drift onto different
trajectories and its passes compare different work; this does not.
"""

import argparse
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--n", type=int, default=1_000_000)
    args = ap.parse_args()
    import torch

    from paper_2511_23030_b200 import _lib
    from paper_2511_23030_b200.workloads import build_c2
    eng = build_c2(args.n, 16, store_dir=tempfile.mkdtemp(prefix="kab_"))
    lib = _lib.load()
    views = []
    for kid in sorted(eng.store.resident_keyframe_ids()):
        kf = eng.store.keyframe_get(kid)
        ids = sorted(eng._visible_for_pose(kf.pose)[0])
        eng.store.ensure_resident(ids)
        slots, n = eng.active.build(eng.store.segments(ids))
        eng.render.ensure(n, kf.intrinsics.width, kf.intrinsics.height)
        views.append((kf, slots, n))

    def sweep(reps):
        for _ in range(reps):
            for kf, slots, n in views:
                eng._device_pass(kf, slots, n, backward=True, adam=False)
        eng.store.slab.grads.zero_()

    sweep(2)   # warm-up (allocations, tile orders)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sweep(args.reps)
    b.record()
    torch.cuda.synchronize()
    passes = args.reps * len(views)
    total = a.elapsed_time(b) / passes
    lib.sm_profile_enable(1)
    _lib.profile_collect()
    sweep(args.reps)
    torch.cuda.synchronize()
    prof = _lib.profile_collect()
    lib.sm_profile_enable(0)
    stages = {k: round(v[0] / passes, 5) for k, v in prof.items() if v[1]}
    # outputs of one pass per view (images, depth, alpha, gradients): equal
    # hashes across builds = bit-identical results
    import hashlib
    h = hashlib.sha1()
    for kf, slots, n in views:
        eng.store.slab.grads.zero_()
        eng._device_pass(kf, slots, n, backward=True, adam=False)
        torch.cuda.synchronize()
        for t in (eng.rgb, eng.depth, eng.alpha, eng.store.slab.grads):
            h.update(t.cpu().numpy().tobytes())
    print(json.dumps({"variant": __import__("os").environ.get("SM_LIB_VARIANT", "main"),
                      "pass_ms": round(total, 5), "passes": passes, "stages_ms": stages,
                      "outputs_sha1": h.hexdigest()[:16],
                      "visible": [n for _, _, n in views]}))


if __name__ == "__main__":
    main()
