"""Host time per FusionPipeline.step against the GPU time (developer tool):
config 3 from pinned host frames; whether the host keeps the GPU fed."""
import sys
import tempfile
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1511_07106_b200 as tf  # noqa: E402
from paper_1511_07106_b200.synth import demo_scene  # noqa: E402

intr = tf.RunConfig().intrinsics()
poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)
scene = demo_scene()
frames = [torch.from_numpy(scene.render_depth(p, intr).data).pin_memory() for p in poses]
cfg = tf.RunConfig(side_length=4.08, resolution=1020, resident_resolution=510, use_groundtruth=True,
                   max_resident=8)
pipe = tf.FusionPipeline(cfg, tempfile.mkdtemp())
for i in range(64):
    pipe.step(frames[i], poses[i])
torch.cuda.synchronize()
host = []
t0 = time.perf_counter()
for i in range(64):
    a = time.perf_counter()
    pipe.step(frames[i], poses[i])
    host.append(time.perf_counter() - a)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
host.sort()
print(f"wall {1e3 * wall / 64:.3f} ms/frame; host step() median {1e3 * host[32]:.3f} ms, "
      f"p90 {1e3 * host[57]:.3f} ms")
