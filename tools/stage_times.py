"""Quick per-stage timing of the C2 mapping step (graph replay + stage events).

    python tools/stage_times.py [--steps 100]

Prints one line per stage (ms per step) and the steady-state step time; used
while optimising kernels (bench.py is the contract-facing benchmark).
"""

import argparse
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--blocks", type=int, default=5)
    ap.add_argument("--no-view-order", action="store_true", help="plain forward tile order (A/B)")
    args = ap.parse_args()
    import torch

    from paper_2511_23030_b200 import _lib
    from paper_2511_23030_b200.workloads import build_c2
    lib = _lib.load()
    eng = build_c2(args.n, 16, store_dir=tempfile.mkdtemp())
    eng.view_tile_order = not args.no_view_order
    eng.warm_graphs()
    for s in range(10):
        eng.optimization_step(0, s)
    torch.cuda.synchronize()
    blocks = []
    for blk in range(args.blocks):   # plain step time: several blocks, median (box noise)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for s in range(args.steps):
            eng.optimization_step(1, blk * args.steps + s)
        b.record()
        torch.cuda.synchronize()
        blocks.append(a.elapsed_time(b) / args.steps)
    plain = sorted(blocks)[len(blocks) // 2]
    # one captured step graph replayed back to back: the device time of a
    # step without the host policy between steps
    g = next(iter(eng._graphs.values()))[0]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(10):
        g.replay()
    a.record()
    for _ in range(args.steps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    graph_only = a.elapsed_time(b) / args.steps
    lib.sm_profile_enable(1)
    eng.drop_graphs()
    eng.warm_graphs()
    _lib.profile_collect()
    eng.reset_counters()
    for s in range(args.steps):
        eng.optimization_step(2, s)
    torch.cuda.synchronize()
    prof = _lib.profile_collect()
    out = {k: round(v[0] / args.steps, 4) for k, v in prof.items() if v[1]}
    out["_sum"] = round(sum(out.values()), 4)
    out["_step_ms"] = round(plain, 4)
    out["_step_ms_min"] = round(min(blocks), 4)
    out["_graph_replay_ms"] = round(graph_only, 4)
    out["_visible"] = eng.counter_gaussians / max(eng.counter_steps, 1)
    out["_instances"] = eng.counter_instances / max(eng.counter_steps, 1)
    ctr = eng.render.ws[:64].view(torch.int32).cpu().numpy()
    out["_big_splats_last"] = int(ctr[5])   # sm_render_counters.reserved[1]: big-splat queue length
    print(json.dumps(out))


if __name__ == "__main__":
    main()
