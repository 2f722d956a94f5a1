"""Helpers to unpack the committed golden fixtures (tests/golden/*.npz)."""
import numpy as np

from paper_2511_23030_b200.core import CameraIntrinsics, Pose


def render_case(g, k):
    it = g[f"c{k}_intr"]
    intr = CameraIntrinsics(fx=float(it[0]), fy=float(it[1]), cx=float(it[2]), cy=float(it[3]),
                            near=float(it[4]), far=float(it[5]), width=int(it[6]), height=int(it[7]))
    scene = dict(positions=g[f"c{k}_positions"], rotations=g[f"c{k}_rotations"],
                 scales=g[f"c{k}_scales"], opacities=g[f"c{k}_opacities"], sh0=g[f"c{k}_sh0"])
    pose = Pose(rotation=g[f"c{k}_pose_q"], translation=g[f"c{k}_pose_t"])
    ref = (g[f"c{k}_rgb"], g[f"c{k}_depth"], g[f"c{k}_alpha"])
    return scene, pose, intr, ref


def oracle_args(scene, pose, intr):
    return (scene["positions"], scene["rotations"], scene["scales"], scene["opacities"],
            scene["sh0"], pose.rotation, pose.translation, intr.fx, intr.fy, intr.cx, intr.cy,
            intr.near, intr.width, intr.height)


def f32(scene):
    return {k: np.asarray(v, dtype=np.float32).astype(np.float64) for k, v in scene.items()}
