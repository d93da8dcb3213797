"""Per-frame cost over the config-3 orbit (developer tool): after one untimed
lap, every orbit frame once with its integrate / update-bracket / general /
exact / raycast times (profile events) and counters."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1511_07106_b200 as tf  # noqa: E402
from paper_1511_07106_b200 import _native as nat  # noqa: E402
from paper_1511_07106_b200.distributed import ShardedFusion  # noqa: E402
from paper_1511_07106_b200.synth import demo_scene  # noqa: E402

intr = tf.RunConfig().intrinsics()
spec = tf.init_grid(4.08, 1020, 510)
params = tf.FusionParams.for_voxel_size(spec.voxel_size)
poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)
scene = demo_scene()
frames = [torch.from_numpy(scene.render_depth(p, intr).data).cuda() for p in poses]
shard = ShardedFusion(spec.keys, spec.voxels_per_side, spec.subvolume_side_length, params, intr)
for i in range(64):
    shard.step(frames[i], poses[i])
torch.cuda.synchronize()
lib = nat.load_library()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
step = [int(a) for a in sys.argv[1:]] or list(range(64))
print("frame  upd_ms  gen_ms  free_ms  exact_ms  ray_ms   updates  exact_vox  swept_gen  coop")
for i in step:
    flush.zero_()
    torch.cuda.synchronize()
    nat.profile_read()
    shard.stats.zero_()
    lib.tf_profile_enable(1)
    shard.step(frames[i], poses[i])
    torch.cuda.synchronize()
    lib.tf_profile_enable(0)
    p = nat.profile_read()
    st = shard.stats.cpu().numpy()
    print(f"{i:5d} {p['integrate_update'][0]:7.3f} {p['integrate_general'][0]:7.3f} {p['integrate_free'][0]:8.3f}"
          f" {p['integrate_exact'][0]:8.3f} {p['raycast'][0]:7.3f} {int(st[nat.STAT_VOXEL_UPDATES]):9d}"
          f" {int(st[nat.STAT_EXACT_VOXELS]):10d} {int(st[nat.STAT_SWEPT_VOXELS]):10d} {int(st[nat.STAT_COOP_RAYS]):5d}")
