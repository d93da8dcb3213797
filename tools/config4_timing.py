"""Where config 4's frame time goes (developer tool): 300 corridor frames
through FusionPipeline.step with host timers around its phases and the GPU
busy time from CUDA events."""
import sys
import time
from pathlib import Path
import tempfile

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1511_07106_b200 as tf  # noqa: E402
from paper_1511_07106_b200 import pipeline as pl  # noqa: E402
from paper_1511_07106_b200.synth import corridor_depth, corridor_scene  # noqa: E402

N = 300
cfg = tf.RunConfig(dynamic=True, block_voxels=258, block_side_length=1.024, max_volumes=16,
                   hysteresis=1.5, max_resident=16, use_groundtruth=True)
intr = cfg.intrinsics()
poses = tf.corridor_trajectory(20.0, 2000)[:N]
scene = corridor_scene()
frames = [torch.from_numpy(corridor_depth(scene, p, intr).data).pin_memory() for p in poses]
timers = {}


def wrap(obj, name):
    fn = getattr(obj, name)

    def w(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        timers[name] = timers.get(name, 0.0) + time.perf_counter() - t0
        return r
    setattr(obj, name, w)


pipe = tf.FusionPipeline(cfg, tempfile.mkdtemp())
for nm in ("_update_placement", "_upload", "_next_map"):
    wrap(pipe, nm)
wrap(pl, "raycast_volumes")
wrap(pipe._integrator.__class__, "__call__") if False else None
orig_int = pipe._integrator


class T:
    def __call__(self, *a, **k):
        t0 = time.perf_counter()
        orig_int(*a, **k)
        timers["integrate"] = timers.get("integrate", 0.0) + time.perf_counter() - t0


pipe._integrator = T()
for i in range(20):
    pipe.step(frames[i], poses[i])
torch.cuda.synchronize()
timers.clear()
from paper_1511_07106_b200 import _native as nat  # noqa: E402
nat.profile_read()
nat.lib().tf_profile_enable(1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for i in range(20, N):
    pipe.step(frames[i], poses[i])
e1.record()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
n = N - 20
print(f"frames {n}: wall {1e3 * wall / n:.3f} ms/frame, gpu events {e0.elapsed_time(e1) / n:.3f} ms/frame")
for k, v in sorted(timers.items(), key=lambda x: -x[1]):
    print(f"  host {k}: {1e3 * v / n:.3f} ms/frame")
nat.lib().tf_profile_enable(0)
prof = nat.profile_read()
for k in ("integrate_all", "integrate_update", "raycast", "raycast_coop"):
    ms, cnt = prof[k]
    print(f"  gpu {k}: {ms / n:.3f} ms/frame ({cnt} launches)")
print("tiles live at end", len(pipe.volumes))
