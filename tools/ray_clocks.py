"""Debug: per-pixel raycast cycle map on the bench workload (config 3)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1511_07106_b200 as tf  # noqa: E402
from paper_1511_07106_b200 import _native as nat  # noqa: E402
from paper_1511_07106_b200.synth import demo_scene  # noqa: E402

intr = tf.RunConfig().intrinsics()
spec = tf.init_grid(4.08, 1020, 510)
params = tf.FusionParams.for_voxel_size(spec.voxel_size)
tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
scene = demo_scene()
poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)
for p in poses[:40]:
    tf.integrate_volumes(tiles, scene.render_depth(p, intr), p, intr, params)
lib = nat.load_library()
clk = torch.zeros(12 * intr.height * intr.width, dtype=torch.int64, device="cuda")
import os  # noqa: E402
if os.environ.get("RAY_CLOCKS_OFF"):  # profile the production kernel (no debug stores)
    rm = tf.RayMap.empty(intr)
    tf.raycast_volumes(tiles, poses[41], intr, rm, params)
    torch.cuda.synchronize()
    sys.exit(0)
lib.tf_debug_ray_clock_buffer(clk.data_ptr())
rm = tf.RayMap.empty(intr)
st = torch.zeros(nat.STAT_COUNT, dtype=torch.int64, device="cuda")
tf.raycast_volumes(tiles, poses[41], intr, rm, params, st)
torch.cuda.synchronize()
lib.tf_debug_ray_clock_buffer(None)
stride = int(os.environ.get("RAY_CLOCKS_STRIDE", "12"))  # 4 for libraries before the diag slots
allc = clk.cpu().numpy()[: stride * intr.height * intr.width].reshape(intr.height, intr.width, stride)
allc = np.concatenate([allc, np.zeros(allc.shape[:2] + (12 - stride,), allc.dtype)], -1).astype(np.float64)
c = allc[..., 0]
smp, ex, summ = allc[..., 1], allc[..., 2], allc[..., 3]
ev = smp - summ
print("per ray: samples %.0f evaluated %.0f exact %.1f summary %.0f" % (smp.mean(), ev.mean(), ex.mean(), summ.mean()))
wmax = lambda a: a.reshape(intr.height // 4, 4, intr.width // 8, 8).max(axis=(1, 3))
print("warp-max evaluated samples mean %.0f (lane mean %.0f); warp cycles / warp-max evaluated = %.0f" % (
    wmax(ev).mean(), ev.mean(), (wmax(c) / np.maximum(wmax(ev), 1)).mean()))
print("cycles per evaluated sample (pixel): median %.0f" % np.median(c / np.maximum(ev, 1)))
hit = np.isfinite(rm.distance)
print("cycles/pixel: mean %.0f median %.0f p90 %.0f max %.0f" % (c.mean(), np.median(c), np.percentile(c, 90), c.max()))
print("hit pixels mean %.0f, miss pixels mean %.0f, hit frac %.2f" % (c[hit].mean(), c[~hit].mean(), hit.mean()))
w = c.reshape(intr.height // 4, 4, intr.width // 8, 8).max(axis=(1, 3))
print("warp max mean %.0f; sum of warp max %.3g vs sum of pixel %.3g" % (w.mean(), w.sum() * 32, c.sum()))
rows = c.reshape(12, 40, 640).mean(axis=(1, 2))
print("row-band means:", " ".join("%.0f" % r for r in rows))
print("stats: samples %d exact %d summary %d" % (st[nat.STAT_RAY_SAMPLES], st[nat.STAT_EXACT_SAMPLES], st[nat.STAT_SUMMARY_SAMPLES]))
dg = allc[..., 4:]
if dg.any():  # diagnostics build (-DTF_RAY_DIAG): cycles / calls per march phase
    names = ["region_at", "cert_sample", "scan", "march_fast"]
    for i, nm in enumerate(names):
        print("  %-12s mean cycles %9.0f calls %7.1f -> %6.0f cycles/call" % (
            nm, dg[..., i].mean(), dg[..., i + 4].mean(), dg[..., i].sum() / max(dg[..., i + 4].sum(), 1)))
np.save("gpurun_out/ray_clocks.npy", allc)
w = np.unravel_index(np.argmax(c), c.shape)
wy, wx = (w[0] // 4) * 4, (w[1] // 8) * 8
print("slowest warp at rows %d-%d cols %d-%d: %.0f cycles; per lane (samples, exact, summary):" % (
    wy, wy + 3, wx, wx + 7, c[w]))
for yy in range(wy, wy + 4):
    print("  ", " ".join("(%d,%d,%d)" % tuple(allc[yy, xx, 1:4]) for xx in range(wx, wx + 8)))
if dg.any():
    for i, nm in enumerate(["region_at", "cert_sample", "scan", "march_fast"]):
        blk = dg[wy:wy + 4, wx:wx + 8]
        print("  slow warp %-12s cycles/lane %9.0f calls/lane %6.1f" % (nm, blk[..., i].mean(), blk[..., i + 4].mean()))
print("  distances:", rm.distance[wy:wy + 4, wx:wx + 8].round(3).tolist())

if os.environ.get("RAY_LANE0"):
    # the same frame with only lane 0 of each warp tracing: lane 0's cycles
    # alone vs. inside its full warp measure the cost of lane divergence
    clk.zero_()
    lib.tf_debug_ray_clock_buffer(clk.data_ptr())
    lib.tf_set_debug_flags(nat.DEBUG_LANE0_ONLY)
    rm2 = tf.RayMap.empty(intr)
    tf.raycast_volumes(tiles, poses[41], intr, rm2, params)
    torch.cuda.synchronize()
    lib.tf_set_debug_flags(0)
    lib.tf_debug_ray_clock_buffer(None)
    solo = clk.cpu().numpy()[: stride * intr.height * intr.width].reshape(intr.height, intr.width, stride)
    full0 = c[0::4, 0::8]
    solo0 = solo[0::4, 0::8, 0].astype(np.float64)
    print("lane 0: mean cycles in full warp %.0f, alone %.0f" % (full0.mean(), solo0.mean()))
    order = np.argsort(full0.ravel())[::-1][:8]
    print("slowest warps, lane-0 cycles full vs alone:",
          " ".join("%.2fM/%.2fM" % (full0.ravel()[i] / 1e6, solo0.ravel()[i] / 1e6) for i in order))

if not os.environ.get("RAY_LANE0") and allc[..., 5].any():
    # timeline of warps (lane 0 of each 8x4 tile): start / end on the global timer
    st0 = allc[0::4, 0::8, 4].ravel()
    en0 = allc[0::4, 0::8, 5].ravel()
    t0 = st0.min()
    st0, en0 = (st0 - t0) / 1e3, (en0 - t0) / 1e3  # microseconds
    T = en0.max()
    grid = np.linspace(0, T, 400)
    active = np.array([((st0 <= t) & (en0 > t)).sum() for t in grid])
    print("kernel %.0f us; warps active (of 2960 slots): " % T +
          " ".join("%d%%:%d" % (p, active[int(p / 100 * 399)]) for p in (10, 30, 50, 70, 80, 90, 95, 99)))
    dur = en0 - st0
    late = np.argsort(en0)[-5:]
    print("last warps to finish: start/dur us", [(round(st0[i]), round(dur[i])) for i in late])
    print("time with < 50%% of slots busy: %.0f us" % ((active < 1480).mean() * T))
