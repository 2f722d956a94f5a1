"""cProfile of the host side of the C2 mapping step (graph replay mode).

    python tools/host_profile.py [--steps 300]
"""

import argparse
import cProfile
import pstats
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    args = ap.parse_args()
    import torch

    from paper_2511_23030_b200.workloads import build_c2
    eng = build_c2(1_000_000, 16, store_dir=tempfile.mkdtemp())
    eng.warm_graphs()
    for s in range(20):
        eng.optimization_step(0, s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(args.steps):
        eng.optimization_step(1, s)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / args.steps
    pr = cProfile.Profile()
    pr.enable()
    for s in range(args.steps):
        eng.optimization_step(2, s)
    pr.disable()
    print(f"wall per step {wall * 1e3:.3f} ms")
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
