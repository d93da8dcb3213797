import sys, tempfile
sys.path.insert(0, '.')
import torch
import paper_1511_07106_b200 as tf
from paper_1511_07106_b200.volumes import VolumeSet
n = 512
params = tf.FusionParams.for_voxel_size(0.002)
for tier in ("host", "host_packed"):
    vset = VolumeSet(params, voxels_per_side=n, voxel_size=0.002, max_resident=2,
                     spill_dir=tempfile.mkdtemp(), spill_tier=tier)
    for k in range(4):
        vset.add((k * 510, 0, 0))
    for f in range(3):
        for k in vset.keys():
            t = vset.acquire(k)
            vset.release(k)
            torch.cuda.synchronize()
            print(tier, f, k, round(torch.cuda.memory_allocated() / 1e9, 2), flush=True)
    del vset, t
    torch.cuda.synchronize()
    print("after del", round(torch.cuda.memory_allocated() / 1e9, 2))
