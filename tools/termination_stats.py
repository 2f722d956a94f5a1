"""Diagnostics: how far into each tile's instance list compositing gets.

    python tools/termination_stats.py

For a few C2 keyframes: instances per tile, fraction of the list before the
block's last contributor (the forward's early-termination horizon), and the
per-pixel contributor position distribution.
"""

import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import ctypes

    import torch

    from paper_2511_23030_b200 import _lib
    from paper_2511_23030_b200.renderloss import camera_for
    from paper_2511_23030_b200.workloads import build_c2
    eng = build_c2(1_000_000, 16, store_dir=tempfile.mkdtemp())
    lib = _lib.load()
    for kid in range(0, 16, 4):
        kf = eng.store.keyframe_get(kid)
        ids = sorted(eng._visible_for_pose(kf.pose)[0])
        slots, n = eng.active.build(eng.store.segments(ids))
        cam = camera_for(kf.pose, kf.intrinsics)
        eng.render.forward(eng.store.slab.params, slots, n, cam, eng.rgb, eng.depth, eng.alpha)
        torch.cuda.synchronize()
        # workspace layout offsets are private to the library; re-derive via sizes
        d = eng.render.dims
        ws = eng.render.ws
        W, H = d.width, d.height
        tiles = ((W + 15) // 16) * ((H + 15) // 16)
        # counters + ranges + pix_last located through a debug copy of the layout
        lay = layout(d)
        ranges = ws[lay["ranges"]:lay["ranges"] + tiles * 8].view(torch.int32).cpu().numpy().reshape(-1, 2)
        last = ws[lay["pix_last"]:lay["pix_last"] + W * H * 4].view(torch.int32).cpu().numpy().reshape(H, W)
        cnt = ranges[:, 1] - ranges[:, 0]
        tl = np.full(tiles, -1)
        for ty in range((H + 15) // 16):
            for tx in range((W + 15) // 16):
                blk = last[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16]
                tl[ty * ((W + 15) // 16) + tx] = blk.max()
        frac = np.where(cnt > 0, (tl - ranges[:, 0] + 1) / np.maximum(cnt, 1), 0)
        T = ws[lay["pix_t"]:lay["pix_t"] + W * H * 4].view(torch.float32).cpu().numpy().reshape(H, W)
        tx_n = (W + 15) // 16
        undone = np.zeros(tiles, int)
        for t in range(tiles):
            ty, tx = divmod(t, tx_n)
            undone[t] = int((T[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] >= 1e-10).sum())
        alive = undone > 0
        fwd_work = np.where(alive, cnt, frac * cnt).sum() / cnt.sum()
        print(f"kf {kid}: n={n} inst={cnt.sum()} per-tile mean={cnt.mean():.0f} max={cnt.max()} "
              f"horizon frac mean={frac[cnt > 0].mean():.3f} (instance-weighted "
              f"{(frac * cnt).sum() / cnt.sum():.3f}); tiles with undone px {alive.mean():.2f}, "
              f"median undone px {np.median(undone[alive]) if alive.any() else 0}, fwd list "
              f"fraction processed {fwd_work:.3f}")


def layout(d):
    """Mirror of render_layout() offsets (csrc/render_fwd.cu) for diagnostics."""
    G = max(d.max_gaussians, 1)
    I = max(d.max_instances, 1)
    W, H = d.width, d.height
    tiles = ((W + 15) // 16) * ((H + 15) // 16)
    npx = W * H
    off = 0
    out = {}

    def take(name, nbytes):
        nonlocal off
        out[name] = off
        off += (max(nbytes, 1) + 255) // 256 * 256

    take("ctr", 64)
    take("rec", G * 64)
    take("rec_sorted", G * 64)
    take("p64", G * 40)
    take("dkey0", G * 8)
    take("dkey1", G * 8)
    take("order0", G * 4)
    take("order1", G * 4)
    take("tcount", G * 4)
    take("tcount_r", G * 4)
    take("toff", G * 4)
    take("ikey0", I * 4)
    take("ikey1", I * 4)
    take("ranges", tiles * 8)
    take("pix_cd", npx * 16)
    take("pix_t", npx * 4)
    take("pix_tlast", npx * 4)
    take("pix_last", npx * 4)
    return out


if __name__ == "__main__":
    main()
