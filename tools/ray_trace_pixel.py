"""Debug: classify the lattice samples along one pixel's ray (config 3 state
of tools/ray_clocks.py) — run-length encoded as
  U unobserved/invalid, G >= 0.99 tau (free), N |v| < 0.99 tau (near), B <= -0.99 tau."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1511_07106_b200 as tf  # noqa: E402
from paper_1511_07106_b200.synth import demo_scene  # noqa: E402

px, py = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (170, 226)
intr = tf.RunConfig().intrinsics()
spec = tf.init_grid(4.08, 1020, 510)
params = tf.FusionParams.for_voxel_size(spec.voxel_size)
tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
scene = demo_scene()
poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)
for p in poses[:40]:
    tf.integrate_volumes(tiles, scene.render_depth(p, intr), p, intr, params)
pose = poses[41]
d = pose.rotation @ np.array([(px - intr.cx) / intr.fx, (py - intr.cy) / intr.fy, 1.0])
d /= np.linalg.norm(d)
o = pose.translation
tau = params.truncation
vs = spec.voxel_size
host = [(np.asarray(t.origin_voxel), t.tsdf, t.weight) for t in tiles]
n = spec.voxels_per_side
codes = []
for k in range(0, 2200):
    q = (o + k * vs * d) / vs
    c = "U"
    for ht, ts, w in host:
        loc = q - ht
        i = np.floor(loc).astype(int)
        if np.any(i < 0) or np.any(i > n - 2):
            continue
        f = loc - i
        ws = w[i[2]:i[2] + 2, i[1]:i[1] + 2, i[0]:i[0] + 2]
        if ws.min() <= 0:
            continue
        t = ts[i[2]:i[2] + 2, i[1]:i[1] + 2, i[0]:i[0] + 2].astype(np.float64)
        v = (t[:, :, 0] * (1 - f[0]) + t[:, :, 1] * f[0])
        v = v[:, 0] * (1 - f[1]) + v[:, 1] * f[1]
        v = v[0] * (1 - f[2]) + v[1] * f[2]
        c = "G" if v >= 0.99 * tau else ("N" if v > -0.99 * tau else "B")
        break
    codes.append(c)
runs = []
for c in codes:
    if runs and runs[-1][0] == c:
        runs[-1][1] += 1
    else:
        runs.append([c, 1])
print("pixel", px, py, "ray dir", d.round(4), "origin", o.round(3))
print(" ".join(f"{c}{n}" for c, n in runs))
