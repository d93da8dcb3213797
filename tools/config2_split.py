"""Config 2's frame split (developer tool): device time of integrate / raycast
(profile events) and the wall time of track() (which ends with its one
read-back) over 63 tracked frames."""
import sys
import tempfile
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1511_07106_b200 as tf  # noqa: E402
from paper_1511_07106_b200 import _native as nat  # noqa: E402
from paper_1511_07106_b200 import pipeline as pl  # noqa: E402
from paper_1511_07106_b200.synth import demo_scene  # noqa: E402

cfg = tf.RunConfig(side_length=3.0, resolution=254, resident_resolution=254, use_groundtruth=False)
intr = cfg.intrinsics()
poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 240)[:64]
scene = demo_scene()
frames = [torch.from_numpy(scene.render_depth(p, intr).data).cuda() for p in poses]
for rep in range(2):
    pipe = tf.FusionPipeline(cfg, tempfile.mkdtemp())
    pipe.step(frames[0], poses[0])
    torch.cuda.synchronize()
    t_track = [0.0]
    real = pl.track

    def timed(*a, **k):
        t0 = time.perf_counter()
        r = real(*a, **k)
        t_track[0] += time.perf_counter() - t0
        return r
    pl.track = timed
    nat.profile_read()
    nat.lib().tf_profile_enable(1)
    t0 = time.perf_counter()
    for i in range(1, 64):
        pipe.step(frames[i])
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    nat.lib().tf_profile_enable(0)
    pl.track = real
    p = nat.profile_read()
    n = 63
    print(f"rep {rep}: {n / sec:.1f} fps, {1e3 * sec / n:.3f} ms/frame; track (wall, incl. its read-back) "
          f"{1e3 * t_track[0] / n:.3f}; integrate {p['integrate_all'][0] / n:.3f}; raycast {p['raycast'][0] / n:.3f} ms")
