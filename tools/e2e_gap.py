"""Step time of the C2 mapping loop with and without the per-step keyframe
upload (bench.py's e2e mode), interleaved blocks in one process.

    python tools/e2e_gap.py [--steps 300] [--blocks 4]
"""
import argparse
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--blocks", type=int, default=4)
    ap.add_argument("--serial-upload", action="store_true", help="upload on the compute stream (A/B)")
    args = ap.parse_args()
    import torch

    from paper_2511_23030_b200.workloads import build_c2
    eng = build_c2(1_000_000, 16, store_dir=tempfile.mkdtemp())
    eng.upload_side_stream = not args.serial_upload
    out = {False: [], True: []}
    for up in (False, True):
        eng.upload_keyframes_each_step = up
        eng.warm_graphs()
    s = 0
    for blk in range(args.blocks):
        for up in (False, True):
            eng.upload_keyframes_each_step = up
            for _ in range(20):
                eng.optimization_step(1, s)
                s += 1
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.steps):
                eng.optimization_step(1, s)
                s += 1
            b.record()
            torch.cuda.synchronize()
            out[up].append(round(a.elapsed_time(b) / args.steps, 4))
    print(json.dumps({"device_ms": out[False], "e2e_ms": out[True], "speculative": eng.counter_speculative}))


if __name__ == "__main__":
    main()
