"""Diagnostic: backward error of the full-size C4 view against the fp64 oracle,
per parameter group, and where the largest opacity errors sit."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from tests.test_render_gpu import _gpu_backward, oracle_args  # noqa: E402


def run(scene, pose, intr, tag):
    from paper_2511_23030_b200.core import quat_to_matrix
    rng = np.random.default_rng(4)
    h, w = intr.height, intr.width
    d_rgb = rng.normal(size=(h, w, 3))
    d_depth = rng.normal(size=(h, w)) * 0.1
    gref = O.render_backward(*oracle_args(scene, pose, intr), d_rgb=d_rgb, d_depth=d_depth)
    gpu = _gpu_backward(scene, pose, intr, d_rgb, d_depth, None)
    print(tag, {k: float(np.linalg.norm(gpu[k] - gref[k]) / max(np.linalg.norm(gref[k]), 1e-30)) for k in gref})
    # rgb-only and depth-only
    for name, dr, dd in (("rgb-only", d_rgb, None), ("depth-only", None, d_depth)):
        gr = O.render_backward(*oracle_args(scene, pose, intr), d_rgb=dr, d_depth=dd)
        gg = _gpu_backward(scene, pose, intr, dr, dd, None)
        print("  ", name, {k: float(np.linalg.norm(gg[k] - gr[k]) / max(np.linalg.norm(gr[k]), 1e-30)) for k in gr})
    e = np.abs(gpu["opacities"] - gref["opacities"])
    top = np.argsort(e)[::-1][:12]
    R = quat_to_matrix(pose.rotation)
    pc = (scene["positions"] - pose.translation) @ R
    for i in top:
        z = pc[i, 2]
        u = intr.fx * pc[i, 0] / z + intr.cx
        v = intr.fy * pc[i, 1] / z + intr.cy
        print(f"   splat {i}: err {e[i]:.3e} ref {gref['opacities'][i]:.4e} gpu {gpu['opacities'][i]:.4e} "
              f"z {z:.2f} uv ({u:.1f},{v:.1f}) op {scene['opacities'][i]:.3f} scale {scene['scales'][i]}")
    # error mass by region
    z = pc[:, 2]
    ok = z > 0.1
    u = np.where(ok, intr.fx * pc[:, 0] / np.where(ok, z, 1) + intr.cx, -1e9)
    v = np.where(ok, intr.fy * pc[:, 1] / np.where(ok, z, 1) + intr.cy, -1e9)
    for name, m in (("last tile row", v >= (intr.height // 16) * 16 - 8),
                    ("last tile col", u >= (intr.width // 16) * 16 - 8),
                    ("near z<2", ok & (z < 2)), ("rest", ok)):
        print(f"   {name}: err^2 share {float((e[m] ** 2).sum() / (e ** 2).sum()):.3f}  n {int(m.sum())}")


def main():
    from paper_2511_23030_b200.core import CameraIntrinsics
    from paper_2511_23030_b200.synthetic import C4_INTR, corridor_poses, corridor_scene
    sc = corridor_scene(1_200_000, length=60.0, seed=7)
    pose = corridor_poses(10, spacing=1.0)[3]
    scene = dict(positions=sc.positions, rotations=sc.rotations, scales=sc.scales,
                 opacities=sc.opacities, sh0=sc.sh0)
    run(scene, pose, C4_INTR, "c4 1241x376")
    from paper_2511_23030_b200.core import quat_to_matrix
    z = ((scene["positions"] - pose.translation) @ quat_to_matrix(pose.rotation))[:, 2]
    for zmin in (0.2, 0.5, 1.0):
        keep = ~((z > 0) & (z < zmin))
        sub = {k: v[keep] for k, v in scene.items()}
        run(sub, pose, C4_INTR, f"c4 without splats at z < {zmin} ({int((~keep).sum())} removed)")


if __name__ == "__main__":
    main()
