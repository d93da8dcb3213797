"""Where does the end-to-end step lose time against the device-timed step?

    python tools/e2e_probe.py

Times 50 config-3 steps (wall clock, one sync at the end) through
FusionPipeline with pinned host frames (the bench's e2e path), FusionPipeline
with device-resident frames, ShardedFusion with device-resident frames and
ShardedFusion with a manual pinned upload, and prints ray / integrate counters
per frame for each (a configuration difference shows up there).
"""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1511_07106_b200 as tf  # noqa: E402
from paper_1511_07106_b200 import _native as nat  # noqa: E402
from paper_1511_07106_b200.distributed import ShardedFusion  # noqa: E402


def run(name, step, stats, n=50, warm=5, frames=64):
    for i in range(warm):
        step(i % frames)
    torch.cuda.synchronize()
    stats.zero_()
    t0 = time.perf_counter()
    for s in range(n):
        step((warm + s) % frames)
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t0) / n
    st = stats.cpu().numpy()
    print(f"{name:34s} {ms:7.3f} ms/step  updates/f={st[nat.STAT_VOXEL_UPDATES] / n:11.0f} "
          f"samples/f={st[nat.STAT_RAY_SAMPLES] / n:11.0f} summary/f={st[nat.STAT_SUMMARY_SAMPLES] / n:11.0f} "
          f"coop/f={st[nat.STAT_COOP_RAYS] / n:6.1f}", flush=True)


def main():
    intr, spec, params, poses, scene = bench.workload(64)
    host = [scene.render_depth(p, intr).data for p in poses]
    pinned = [torch.from_numpy(f).pin_memory() for f in host]
    dev = [f.cuda() for f in pinned]
    cfg = tf.RunConfig(side_length=4.08, resolution=1020, resident_resolution=510,
                       use_groundtruth=True, max_resident=8)
    pipe = tf.FusionPipeline(cfg, tempfile.mkdtemp())
    res = torch.empty(pipe.stats.shape, dtype=pipe.stats.dtype).pin_memory()

    def pipe_pinned(i):
        pipe.step(pinned[i], poses[i])
        res.copy_(pipe.stats, non_blocking=True)
    run("FusionPipeline, pinned frames", pipe_pinned, pipe.stats)

    def pipe_dev(i):
        pipe.step(dev[i], poses[i])
    run("FusionPipeline, device frames", pipe_dev, pipe.stats)
    del pipe
    torch.cuda.empty_cache()

    shard = ShardedFusion(spec.keys, spec.voxels_per_side, spec.subvolume_side_length, params, intr)

    def shard_dev(i):
        shard.step(dev[i], poses[i])
    run("ShardedFusion, device frames", shard_dev, shard.stats)
    buf = torch.empty_like(dev[0])

    def shard_pinned(i):
        buf.copy_(pinned[i], non_blocking=True)
        shard.step(buf, poses[i])
    run("ShardedFusion, pinned upload", shard_pinned, shard.stats)


if __name__ == "__main__":
    main()
