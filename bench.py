"""Benchmark: TSDF voxel-updates/s and frames/s of the multi-volume mapper.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], the configuration the metric is quoted
on "at 1/2/4/8 B200"): 8 fixed 512^3 volumes tiling a 4.08 m cube at 4 mm
(init_grid(4.08, 1020, 510)), 640x480 frames of the demo scene (sphere +
floor + box) along orbit_trajectory((0,0,1.5), 1.5, 64), ground-truth poses.
One step = one frame through the hot path: fused integration of every
volume + fused raycast of every volume (+ all-gather / _hit_wins merge of
the partial ray maps across ranks when N > 1).  With N GPUs the 8 volumes
are owned by the ranks in checkerboard-spread chunks (total work fixed -> "strong").

value  = voxel updates per frame x frames/s, inputs resident in HBM, CUDA
         events on the launching stream, L2 flushed (256 MiB write) between
         timed steps, max over ranks.
e2e    = the same through the public FusionPipeline.step API with the frame
         read from pinned host memory each step (H2D inside the timed region)
         and the step's counters read back (D2H).
config2 (secondary): BASELINE configs[1] — one 256^3 volume with ICP
         tracking on (integrate + raycast + projective ICP per frame).

--impl reference times the reference algorithm on the host CPU (the C
restatement in oracle/, all host threads) on the same workload and metric.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "TSDF voxel-updates/sec and frames/sec at 1/2/4/8 B200; % HBM roofline"
BYTES_PER_UPDATE = 16  # read + write of f32 tsdf and f32 weight
FALLBACK_HBM_GBS = 6650.0


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-color", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-config2", action="store_true")
    p.add_argument("--frames", type=int, default=64, help="distinct frames cycled through")
    return p.parse_args()


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def workload(nframes: int):
    import paper_1511_07106_b200 as tf
    from paper_1511_07106_b200.synth import demo_scene

    intr = tf.RunConfig().intrinsics()
    spec = tf.init_grid(4.08, 1020, 510)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 64)[:nframes]
    scene = demo_scene()
    return intr, spec, params, poses, scene


def config_desc(n_gpus: int) -> dict:
    return {"workload": "configs[2]: 8 fixed 512^3 TSDF volumes at 4 mm (init_grid(4.08, 1020, "
                        "510)), 640x480 demo-scene orbit frames, ground-truth poses; step = "
                        "integrate + raycast of every volume",
            "volumes": 8, "voxels_per_side": 512, "voxel_size_m": 0.004, "image": "640x480",
            "ownership": f"checkerboard-spread chunks over {n_gpus} rank(s) (distributed.owned_keys)",
            "l2": "flushed between timed steps (256 MiB write); volumes 8.6 GB > L2"}


def peak_hbm() -> tuple[float, str]:
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            return float(json.loads(f.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int) -> None:
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self._t.join(timeout=2)

    def summary(self) -> dict | None:
        rows = []
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) == 6:
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[2:]))
                except ValueError:
                    pass
        if not rows:
            return None
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        active = sorted({names[i] for _, _, flags in rows for i, f in enumerate(flags)
                         if f.lower().startswith("active")})
        return {"sm_mhz": statistics.median(r[0] for r in rows),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": active, "samples": len(rows)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TFB200_BENCH_FUNCTIONAL=1: every rank on cuda:0 over gloo — a functional
    # check of the N > 1 path on a one-GPU box; its timings mean nothing
    functional = os.environ.get("TFB200_BENCH_FUNCTIONAL") == "1"
    if functional:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1511_07106_b200 as tf
    from paper_1511_07106_b200 import _native as nat
    from paper_1511_07106_b200.distributed import ShardedFusion, broadcast_frame

    lib = nat.load_library()
    intr, spec, params, poses, scene = workload(args.frames)
    nframes = len(poses)
    host_frames = [scene.render_depth(p, intr).data for p in poses]
    dev_frames = torch.stack([torch.from_numpy(f) for f in host_frames]).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: int) -> int:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.int64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return int(t.item())

    shard = ShardedFusion(spec.keys, spec.voxels_per_side, spec.subvolume_side_length, params,
                          intr, rank, world)

    # ---- warm-up (also the per-frame work cycle starts here) ----
    for i in range(args.warmup):
        shard.step(dev_frames[i % nframes], poses[i % nframes])
    barrier()
    if shard._peer is not None and shard._peer.error():
        raise RuntimeError("peer-memory ray-map reduction: a flag wait timed out (warm-up)")

    # ---- timed region: resident inputs, per-step events, L2 flushed between ----
    shard.stats.zero_()
    nat.profile_read()  # drop warm-up records
    lib.tf_profile_enable(1)
    launches0 = lib.tf_launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stops = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        barrier()
        for s in range(args.steps):
            flush.zero_()
            i = (args.warmup + s) % nframes
            starts[s].record()
            shard.step(dev_frames[i], poses[i])
            stops[s].record()
        barrier()
    lib.tf_profile_enable(0)
    launches = lib.tf_launch_count() - launches0
    if shard._peer is not None and shard._peer.error():
        raise RuntimeError("peer-memory ray-map reduction: a flag wait timed out")
    ms_total = sum(a.elapsed_time(b) for a, b in zip(starts, stops))
    prof = nat.profile_read()
    st = shard.stats.cpu().numpy()
    updates_local = int(st[nat.STAT_VOXEL_UPDATES])
    ms_total = max_over_ranks(ms_total)
    updates = sum_over_ranks(updates_local)
    samples = sum_over_ranks(int(st[nat.STAT_RAY_SAMPLES]))
    ms_per_step = ms_total / args.steps
    fps = 1000.0 / ms_per_step
    updates_per_frame = updates / args.steps
    value = updates_per_frame * fps

    # roofline of the dominant kernel (the voxel-update kernel), this rank
    upd_ms, upd_launches = prof["integrate_update"]
    int_ms, _ = prof["integrate_all"]
    ray_ms, ray_launches = prof["raycast"]
    peak, peak_src = peak_hbm()
    achieved = (BYTES_PER_UPDATE * updates_local / max(upd_launches, 1)) / (
        upd_ms / max(upd_launches, 1) / 1e3) / 1e9 if upd_ms > 0 else 0.0
    traffic = ray_traffic = None
    tfile = ROOT / "profiles" / "traffic_r01.json"
    if tfile.exists():
        try:
            tj = json.loads(tfile.read_text())
            traffic = tj.get("integrate_update_bracket_bytes_per_launch")
            ray_traffic = next((v for k, v in tj.get("per_kernel_dram_bytes", {}).items()
                                if k.startswith("raycast_kernel")), None)
        except Exception:
            traffic = ray_traffic = None
    # raycast: not HBM-bound (gathers mostly hit L1/L2); reported
    # against the same HBM peak for scale, with the nominal 64 B per evaluated
    # (gathering) sample: certified-free samples read no voxels
    evaluated = samples - sum_over_ranks(int(st[nat.STAT_SUMMARY_SAMPLES]))
    ray_achieved = (64.0 * evaluated / max(ray_launches, 1)) / (ray_ms / max(ray_launches, 1) / 1e3) / 1e9 \
        if ray_ms > 0 else 0.0

    # per-kernel sub-rooflines of the update bracket (16 B per update each)
    def comp(kind, n_updates):
        ms, n = prof[kind]
        if ms <= 0:
            return None
        gbs = BYTES_PER_UPDATE * n_updates / (ms / 1e3) / 1e9
        return {"ms_per_launch": ms / max(n, 1), "updates_per_launch": n_updates / max(n, 1),
                "achieved_gbs": gbs, "frac": gbs / peak if peak else None}
    free_upd = int(st[nat.STAT_FREE_KERNEL_UPDATES])
    exact_upd = int(st[nat.STAT_EXACT_UPDATES])
    components = {
        "brick_free_kernel (certified free-space bricks, bandwidth-bound)": comp("integrate_free", free_upd),
        "brick_update_kernel (general bricks: float32 screen + exact FP64 update)":
            comp("integrate_general", updates_local - free_upd - exact_upd),
        "exact_queue_kernel (near-surface band, reference arithmetic)": comp("integrate_exact", exact_upd),
    }

    result = {
        "metric": METRIC, "value": value, "unit": "voxel-updates/s",
        "frames_per_s": fps, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(config_desc(world), **({"raymap_exchange": {
            "p2p": "peer-memory reduce kernel (csrc/comm.cu, CUDA IPC over NVLink)",
            "collective": "NCCL row-block all-to-all + merge + all-gather"}[shard.exchange]}
            if world > 1 else {})),
        "voxel_updates_per_frame": updates_per_frame,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "kernel": "integrate update bracket (brick_update_kernel + brick_free_kernel + "
                               "exact_queue_kernel, TF_PROF_INTEGRATE_UPDATE)", "peak_source": peak_src,
                     "bytes_per_update": BYTES_PER_UPDATE,
                     "launches": upd_launches, "kernel_ms_per_launch": upd_ms / max(upd_launches, 1),
                     "updates_per_launch": updates_local / max(upd_launches, 1),
                     "components": components},
        "roofline_raycast": {"bound": "latency (dependent gathers, divergence); not hbm",
                             "achieved": ray_achieved, "peak": peak, "unit": "GB/s",
                             "frac": ray_achieved / peak if peak else None, "traffic": ray_traffic,
                             "kernel": "raycast_kernel", "bytes_per_evaluated_sample": 64,
                             "evaluated_samples_per_launch": evaluated / max(ray_launches, 1),
                             "kernel_ms_per_launch": ray_ms / max(ray_launches, 1)},
        "breakdown_ms_per_step": {"integrate_update_kernel": upd_ms / args.steps,
                                  "integrate_total": int_ms / args.steps,
                                  "raycast": ray_ms / args.steps},
        "integrate": {"noop_updates_per_frame": sum_over_ranks(int(st[nat.STAT_NOOP_UPDATES])) / args.steps, "swept_voxels_per_frame": sum_over_ranks(int(st[nat.STAT_SWEPT_VOXELS])) / args.steps,
                      "exact_path_voxels_per_frame": sum_over_ranks(int(st[nat.STAT_EXACT_VOXELS])) / args.steps,
                      "column_rejected_per_frame": sum_over_ranks(int(st[nat.STAT_COL_SKIPPED])) / args.steps,
                      "depth_rejected_per_frame": sum_over_ranks(int(st[nat.STAT_DEPTH_SKIPPED])) / args.steps,
                      "active_bricks_per_frame": sum_over_ranks(int(st[nat.STAT_ACTIVE_BRICKS])) / args.steps,
                      "free_space_bricks_per_frame": sum_over_ranks(int(st[nat.STAT_FREE_BRICKS])) / args.steps,
                      "general_bricks_all_free_per_frame": sum_over_ranks(int(st[nat.STAT_GENERAL_ALL_FREE])) / args.steps,
                      "general_parts_all_free_per_frame": sum_over_ranks(int(st[nat.STAT_PART_ALL_FREE])) / args.steps,
                      "general_parts_all_skip_per_frame": sum_over_ranks(int(st[nat.STAT_PART_ALL_SKIP])) / args.steps,
                      "total_bricks": sum_over_ranks(int(st[nat.STAT_TOTAL_BRICKS])) // max(args.steps, 1)},
        "raycast": {"exact_samples_per_frame": sum_over_ranks(int(st[nat.STAT_EXACT_SAMPLES])) / args.steps,
                    "certification_failures": sum_over_ranks(int(st[nat.STAT_CERT_FAILURES])),
                    "summary_certified_samples_per_frame": sum_over_ranks(int(st[nat.STAT_SUMMARY_SAMPLES])) / args.steps,
                    "samples_per_frame": samples / args.steps,
                    "coop_rays_per_frame": sum_over_ranks(int(st[nat.STAT_COOP_RAYS])) / args.steps,
                    "coop_pass_ms_per_frame": prof["raycast_coop"][0] / args.steps,
                    "samples_per_s": samples / (ms_total / 1e3)},
        "gpu_launches": int(launches),
    }
    cs = clocks.summary()
    result["clocks"] = cs

    # ---- the same step with colour (north_star; the reference has no colour) ----
    if not args.no_color and world == 1:
        result["color"] = run_color(args, tf, torch, spec, params, intr, poses, scene, barrier)

    # ---- e2e through the public pipeline API, frames from pinned host memory ----
    if not args.no_e2e:
        result["e2e"] = run_e2e(args, tf, nat, torch, dist, rank, world, intr, spec, params,
                                poses, host_frames, barrier, max_over_ranks, sum_over_ranks)
    del shard, dev_frames
    torch.cuda.empty_cache()

    if not args.no_config2:
        result["config2"] = run_config2(args, tf, nat, torch, barrier, max_over_ranks)

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(intr, spec, params, poses, host_frames)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_color(args, tf, torch, spec, params, intr, poses, scene, barrier) -> dict:
    """Config 3 with an RGB frame fused into a colour channel per volume (the
    band voxels' running mean, tf_integrate_rgb) and the model colours
    rendered (tf_raycast_colors) every step: device-resident inputs."""
    from paper_1511_07106_b200.distributed import ShardedFusion
    from paper_1511_07106_b200.synth import render_rgb

    steps = args.steps  # the same frame mix as the device-timed loop (early frames are slower)
    n = len(poses)
    depth = [torch.from_numpy(scene.render_depth(p, intr).data).cuda() for p in poses]
    rgb = [torch.from_numpy(render_rgb(scene, p, intr)).cuda() for p in poses]
    shard = ShardedFusion(spec.keys, spec.voxels_per_side, spec.subvolume_side_length, params, intr,
                          color=True)
    for i in range(args.warmup):
        shard.step(depth[i % n], poses[i % n], color=rgb[i % n])
        tf.raycast_colors(shard.tiles, shard.model, poses[i % n], intr)
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in range(steps):
        i = (args.warmup + s) % n
        shard.step(depth[i], poses[i], color=rgb[i])
        tf.raycast_colors(shard.tiles, shard.model, poses[i], intr)
    b.record()
    barrier()
    ms = a.elapsed_time(b) / steps
    del shard
    torch.cuda.empty_cache()
    return {"frames_per_s": 1000.0 / ms, "ms_per_step": ms, "steps": steps,
            "path": "ShardedFusion.step(depth, pose, color=rgb) + raycast_colors, inputs resident",
            "note": "colour is not in the reference; no L2 flush between steps"}


def run_e2e(args, tf, nat, torch, dist, rank, world, intr, spec, params, poses, host_frames,
            barrier, max_over_ranks, sum_over_ranks) -> dict:
    from paper_1511_07106_b200.distributed import ShardedFusion, broadcast_frame

    nframes = len(poses)
    pinned = [torch.from_numpy(f).pin_memory() for f in host_frames]
    steps = args.steps  # the same frame mix as the device-timed loop (early frames are slower)
    if world == 1:
        cfg = tf.RunConfig(side_length=4.08, resolution=1020, resident_resolution=510,
                           use_groundtruth=True, max_resident=8)
        spill = tempfile.mkdtemp(prefix="tfb200_spill_")
        pipe = tf.FusionPipeline(cfg, spill)

        result = torch.empty(pipe.stats.shape, dtype=pipe.stats.dtype).pin_memory()

        def step(i):
            pipe.step(pinned[i], poses[i])          # public API: H2D inside step()
            result.copy_(pipe.stats, non_blocking=True)  # D2H of the step's counters
            return result
    else:
        shard = ShardedFusion(spec.keys, spec.voxels_per_side, spec.subvolume_side_length,
                              params, intr, rank, world)
        # the frame goes up (rank 0) and out (broadcast) on a side stream into
        # one of two buffers, so the next frame's culling can start while this
        # frame's raycast runs (ShardedFusion.step depth_ready)
        bufs = [torch.empty(host_frames[0].shape, dtype=torch.float64, device="cuda") for _ in range(2)]
        side = torch.cuda.Stream()
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        free = [torch.cuda.Event(), torch.cuda.Event()]
        for e in free:
            e.record()

        result = torch.empty(shard.stats.shape, dtype=shard.stats.dtype).pin_memory()

        def step(i):
            slot = i & 1
            side.wait_event(free[slot])
            with torch.cuda.stream(side):
                if rank == 0:
                    bufs[slot].copy_(pinned[i], non_blocking=True)
                broadcast_frame(bufs[slot])
                ready[slot].record(side)
            torch.cuda.current_stream().wait_event(ready[slot])
            shard.step(bufs[slot], poses[i], depth_ready=ready[slot])
            free[slot].record()
            result.copy_(shard.stats, non_blocking=True)
            return result

    for i in range(args.warmup):
        out = step(i % nframes)
    torch.cuda.synchronize()
    barrier()
    before = int(out[nat.STAT_VOXEL_UPDATES])
    # every step uploads its frame from pinned memory and reads its counters
    # back into pinned memory, both stream-ordered; the host does not wait per
    # step, only once at the end (the last read has landed when the clock stops)
    t0 = time.perf_counter()
    for s in range(steps):
        out = step((args.warmup + s) % nframes)
    torch.cuda.synchronize()
    barrier()
    sec = max_over_ranks(time.perf_counter() - t0)
    updates = sum_over_ranks(int(out[nat.STAT_VOXEL_UPDATES]) - before)
    return {"value": updates / sec, "unit": "voxel-updates/s", "frames_per_s": steps / sec,
            "h2d_bytes_per_step": int(host_frames[0].nbytes) if rank == 0 else 0,
            "d2h_bytes_per_step": int(out.numel() * out.element_size()), "steps": steps,
            "path": "FusionPipeline.step(pinned host frame)" if world == 1 else
                    "rank-0 H2D + NCCL broadcast (side stream) + ShardedFusion.step"}


def run_config2(args, tf, nat, torch, barrier, max_over_ranks) -> dict:
    """BASELINE configs[1]: one 256^3 volume, ICP tracking on, 1.5-degree orbit."""
    from paper_1511_07106_b200.synth import demo_scene

    cfg = tf.RunConfig(side_length=3.0, resolution=254, resident_resolution=254,
                       use_groundtruth=False)
    intr = cfg.intrinsics()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 240)[:64]
    scene = demo_scene()
    steps = min(args.steps, 63)
    frames = [torch.from_numpy(scene.render_depth(p, intr).data).cuda() for p in poses[:steps + 1]]
    # an untimed pass over the same frames first (allocator growth, workspaces,
    # first launches), then the timed pass with a fresh pipeline
    warm = tf.FusionPipeline(cfg, tempfile.mkdtemp(prefix="tfb200_c2w_"))
    warm.step(frames[0], poses[0])
    for i in range(1, steps + 1):
        warm.step(frames[i])
    torch.cuda.synchronize()
    del warm
    pipe = tf.FusionPipeline(cfg, tempfile.mkdtemp(prefix="tfb200_c2_"))
    pipe.step(frames[0], poses[0])   # frame 0 defines the world frame
    gc.collect()
    barrier()
    pipe.stats.zero_()
    gc.disable()  # no collector pause inside the 60-80 ms timed pass
    t0 = time.perf_counter()
    for i in range(1, steps + 1):
        pipe.step(frames[i])
        if os.environ.get("TFB200_C2_TRACE"):
            torch.cuda.synchronize()
            print(f"config2 frame {i}: {1e3 * (time.perf_counter() - t0):.2f} ms", file=sys.stderr)
    barrier()
    sec = max_over_ranks(time.perf_counter() - t0)
    gc.enable()
    ks = pipe.kernel_stats()
    lost = sum(1 for r in pipe.records[1:] if not r.tracked)
    err = max(float(np.abs(p.translation - q.translation).max())
              for p, q in zip(pipe.poses, poses[:steps + 1]))
    return {"workload": "configs[1]: one 256^3 volume (init_grid(3.0, 254, 254)), 640x480, "
                        "1.5-degree orbit, ICP tracking on", "frames": steps,
            "frames_per_s": steps / sec, "voxel_updates_per_s": ks["voxel_updates"] / sec,
            "lost_frames": lost, "max_translation_error_m": err}


# ---------------------------------------------------------------------------
# CPU baseline (oracle restatement of the reference kernels, all host threads)
# ---------------------------------------------------------------------------

def cpu_frame_sample(intr, spec, params, poses, host_frames, volumes: int, threads: int,
                     first: int = 0) -> dict:
    import oracle

    n = spec.voxels_per_side
    vs = spec.voxel_size
    coarse = max(2, int(round(0.5 * params.truncation / vs)))
    keys = [spec.keys[(first + i) % len(spec.keys)] for i in range(volumes)]
    tiles = [(np.zeros((n, n, n), np.float32), np.zeros((n, n, n), np.float32)) for _ in keys]
    p0, p1 = poses[0], poses[1]
    for (t, w), k in zip(tiles, keys):
        inv = p0.invert()
        oracle.integrate(t, w, k, vs, host_frames[0], inv.rotation, inv.translation,
                         p0.translation, intr.fx, intr.fy, intr.cx, intr.cy, params.truncation,
                         params.max_weight, params.sample_weight, threads=threads)
    inv = p1.invert()
    t0 = time.perf_counter()
    updates = 0
    for (t, w), k in zip(tiles, keys):
        updates += oracle.integrate(t, w, k, vs, host_frames[1], inv.rotation, inv.translation,
                                    p1.translation, intr.fx, intr.fy, intr.cx, intr.cy,
                                    params.truncation, params.max_weight, params.sample_weight,
                                    threads=threads)
    t_int = time.perf_counter() - t0
    d = np.full((intr.height, intr.width), np.inf)
    v = np.zeros((intr.height, intr.width, 3))
    nn = np.zeros_like(v)
    t0 = time.perf_counter()
    for (t, w), k in zip(tiles, keys):
        oracle.raycast(t, w, k, vs, params.truncation, coarse, p1.rotation, p1.translation,
                       intr.fx, intr.fy, intr.cx, intr.cy, d, v, nn, threads=threads)
    t_ray = time.perf_counter() - t0
    return {"updates": updates, "t_integrate": t_int, "t_raycast": t_ray, "volumes": volumes}


def cpu_baseline(intr, spec, params, poses, host_frames) -> dict:
    import oracle

    threads = oracle.default_threads()
    vols = 8 if threads >= 16 else 2
    s = cpu_frame_sample(intr, spec, params, poses, host_frames, vols, threads)
    frame_s = (s["t_integrate"] + s["t_raycast"]) * 8 / vols
    updates_frame = s["updates"] * 8 / vols
    return {"value": updates_frame / frame_s, "unit": "voxel-updates/s", "cores": threads,
            "kind": "port", "frames_per_s": 1.0 / frame_s,
            "sample": f"frame 1 of the same workload, {vols} of 8 volumes (integrate + raycast, "
                      f"C oracle on {threads} host threads), scaled to 8 volumes",
            "integrate_s_per_volume": s["t_integrate"] / vols,
            "raycast_s_per_volume": s["t_raycast"] / vols}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # the CPU reference runs once, on rank 0
    import oracle

    world = int(os.environ.get("WORLD_SIZE", "1"))
    threads = oracle.default_threads()
    intr, spec, params, poses, scene = workload(2)
    host_frames = [scene.render_depth(p, intr).data for p in poses]
    # exactly --warmup untimed and --steps timed samples; each sample is
    # bounded (volumes per sample shrink as K + W grow: ~120 volume-samples in
    # all, ~0.5 s each) and the samples walk round-robin over the 8 volumes
    steps, warmup = max(1, args.steps), max(0, args.warmup)
    cap = 8 if threads >= 32 else (4 if threads >= 8 else 1)
    vols = max(1, min(cap, 120 // (steps + warmup)))
    for i in range(warmup):
        cpu_frame_sample(intr, spec, params, poses, host_frames, vols, threads, first=i * vols)
    times, ups = [], []
    for i in range(steps):
        s = cpu_frame_sample(intr, spec, params, poses, host_frames, vols, threads,
                             first=(warmup + i) * vols)
        times.append((s["t_integrate"] + s["t_raycast"]) * 8 / vols)
        ups.append(s["updates"] * 8 / vols)
    frame_s = sum(times) / len(times)
    value = (sum(ups) / len(ups)) / frame_s
    sample = (f"per step: frame 1 of the workload on {vols} of the 8 volumes (round-robin over the "
              f"steps; integrate + raycast), C restatement of the reference kernels on {threads} "
              f"host threads, scaled to 8")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "voxel-updates/s",
        "frames_per_s": 1.0 / frame_s, "n_gpus": world, "steps": steps, "warmup": warmup,
        "ms_per_step": frame_s * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_desc(world),
        "cpu_baseline": {"value": value, "unit": "voxel-updates/s", "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "voxel-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def main() -> None:
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
