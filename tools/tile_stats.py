"""Per-tile work distribution of the C2 mapping step (diagnostics).

    python tools/tile_stats.py [--n 1000000] [--keyframes 4]

For a few keyframes: instances per tile, instances the backward revisits
(up to the tile's last contributor) and how concentrated they are -- the
compositing kernels' load balance across the 148 SMs depends on the tail.
"""

import argparse
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--keyframes", type=int, default=4)
    args = ap.parse_args()
    import torch

    from paper_2511_23030_b200 import _lib
    from paper_2511_23030_b200.workloads import build_c2
    lib = _lib.load()
    eng = build_c2(args.n, 16, store_dir=tempfile.mkdtemp())
    r = eng.render
    out = []
    for k in range(args.keyframes):
        eng.optimization_step(k * 5 % 16, k)
        torch.cuda.synchronize()
        d = r.dims
        w, h = d.width, d.height
        tx, ty = (w + 15) // 16, (h + 15) // 16
        o_r = lib.sm_render_ws_offset(d, 0)
        o_l = lib.sm_render_ws_offset(d, 1)
        ws = r.ws
        ranges = ws[o_r:o_r + tx * ty * 8].view(torch.int32).cpu().numpy().view(np.uint32).reshape(-1, 2)
        last = ws[o_l:o_l + w * h * 4].view(torch.int32).cpu().numpy().reshape(h, w)
        lp = np.full((ty * 16, tx * 16), -1, np.int64)
        lp[:h, :w] = last
        maxlast = lp.reshape(ty, 16, tx, 16).max(axis=(1, 3)).reshape(-1)
        L = (ranges[:, 1].astype(np.int64) - ranges[:, 0])
        V = np.where(maxlast >= 0, maxlast - ranges[:, 0].astype(np.int64) + 1, 0)
        srt = np.sort(V)[::-1]
        o_t = lib.sm_render_ws_offset(d, 3)
        cnt = ws[o_t:o_t + 4 * eng.last_n].view(torch.int32).cpu().numpy()
        big = cnt[cnt > 32]
        out.append({
            "keyframe_step": k, "tiles": int(len(L)), "instances": int(L.sum()), "visited": int(V.sum()),
            "L_mean": float(L.mean()), "L_max": int(L.max()), "L_p99": float(np.percentile(L, 99)),
            "V_mean": float(V.mean()), "V_max": int(V.max()), "V_p99": float(np.percentile(V, 99)),
            "V_top10": srt[:10].tolist(),
            "V_max_over_mean": float(V.max() / max(V.mean(), 1)),
            "big_splats": int(len(big)), "big_instances": int(big.sum()),
            "big_max": int(big.max()) if len(big) else 0,
            "big_hist": np.histogram(big, bins=[33, 64, 128, 256, 512, 1024, 4096])[0].tolist(),
        })
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    main()
