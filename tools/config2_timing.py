import sys, time, tempfile
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_1511_07106_b200 as tf
from paper_1511_07106_b200.synth import demo_scene
cfg = tf.RunConfig(side_length=3.0, resolution=254, resident_resolution=254, use_groundtruth=False)
intr = cfg.intrinsics()
poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 240)[:64]
scene = demo_scene()
frames = [torch.from_numpy(scene.render_depth(p, intr).data).cuda() for p in poses]
for rep in range(3):
    pipe = tf.FusionPipeline(cfg, tempfile.mkdtemp())
    pipe.step(frames[0], poses[0])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ts = []
    for i in range(1, 64):
        a = time.perf_counter()
        pipe.step(frames[i])
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - a)
    sec = time.perf_counter() - t0
    ts = np.array(ts) * 1e3
    print("rep %d: %.1f fps; per-frame ms median %.2f p90 %.2f max %.2f" % (rep, 63 / sec, np.median(ts), np.percentile(ts, 90), ts.max()))
