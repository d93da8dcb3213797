import sys, tempfile
sys.path.insert(0, '.')
import torch
import paper_1511_07106_b200 as tf
from paper_1511_07106_b200.synth import demo_scene
cfg = tf.RunConfig(side_length=3.0, resolution=254, resident_resolution=254, use_groundtruth=False)
intr = cfg.intrinsics()
poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 240)[:8]
scene = demo_scene()
frames = [torch.from_numpy(scene.render_depth(p, intr).data).cuda() for p in poses]
pipe = tf.FusionPipeline(cfg, tempfile.mkdtemp())
pipe.step(frames[0], poses[0])
for i in range(1, 8):
    pipe.step(frames[i])
torch.cuda.synchronize()
print("ok")
