"""Benchmark: TSDF voxel-updates/s and frames/s of the multi-volume mapper.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], the configuration the metric is quoted
on "at 1/2/4/8 B200"): 8 fixed 512^3 volumes tiling a 4.08 m cube at 4 mm
(init_grid(4.08, 1020, 510)), 640x480 frames of the demo scene (sphere +
floor + box) along orbit_trajectory((0,0,1.5), 1.5, 64), ground-truth poses.
One step = one frame through the hot path: fused integration of every
volume + fused raycast of every volume (+ the _hit_wins reduction of the
partial ray maps across ranks when N > 1).

Frame schedule (identical in every arm, independent of K): one untimed lap
over the 64 orbit frames builds the map, W warm-up steps follow, then the K
timed steps take frames spread uniformly over the orbit (frame
floor(s * 64 / K) for K <= 64, s mod 64 beyond), so a short run times the
same mix as a long one.

value  = voxel updates per frame x frames/s, inputs resident in HBM, CUDA
         events on the launching stream per step, L2 flushed (256 MiB write)
         between timed steps, max over ranks.
e2e    = the same through the public FusionPipeline.step API with the frame
         read from pinned host memory each step (H2D inside the timed region)
         and the step's counters read back (D2H).
Extra legs (N = 1): config1 / config2 (BASELINE configs[0], [1]) with their
CPU baselines, config4 (dynamic placement over the 2000-frame corridor),
config5 (1024^3 tiles through the pinned-host spill tier), colour.

--impl reference times the reference algorithm on the host CPU on the same
frames and map state: the C restatement in oracle/ on all host threads (the
headline CPU arm) and, as a second stated baseline, the unmodified reference
package (numba, single core) from baseline/_ref on a bounded sample.

--gpus N without a torchrun environment re-launches this script under
torch.distributed.run with N ranks (127.0.0.1); rank 0 prints the line.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import socket
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
LAP = 64               # frames of the orbit (BASELINE configs[0..2])


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=64)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-color", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extra", action="store_true", help="skip the config1/2/4/5 legs")
    p.add_argument("--no-numba", action="store_true", help="reference arm: skip the numba sample")
    p.add_argument("--only", choices=["config1", "config2", "config4", "config5", "scaling_projection"],
                   help="run just this extra leg (debugging)")
    return p.parse_args()


# ---------------------------------------------------------------------------
# launcher
# ---------------------------------------------------------------------------

def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_if_needed(args) -> None:
    """--gpus N > 1 outside torchrun: start N ranks of this script."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None:
        if args.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
                   f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
            sys.exit(subprocess.call(cmd))
        return
    if int(env_world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}")


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def workload():
    import paper_1511_07106_b200 as tf
    from paper_1511_07106_b200.synth import demo_scene

    intr = tf.RunConfig().intrinsics()
    spec = tf.init_grid(4.08, 1020, 510)
    params = tf.FusionParams.for_voxel_size(spec.voxel_size)
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, LAP)
    return intr, spec, params, poses, demo_scene()


def timed_frames(k: int) -> list[int]:
    return [(s * LAP) // k for s in range(k)] if k <= LAP else [s % LAP for s in range(k)]


def warm_frames(w: int) -> list[int]:
    return [(LAP // 2 + s * 7) % LAP for s in range(w)]


SCHEDULE_DESC = ("one untimed lap over the 64 orbit frames, W warm-up frames, then K timed frames "
                 "spread uniformly over the orbit (floor(s*64/K)); identical in both arms")


def config_desc(n_gpus: int, retile: int = 1, mode: str = "volumes") -> dict:
    d = {"workload": "configs[2]: 8 fixed 512^3 TSDF volumes at 4 mm (init_grid(4.08, 1020, 510)), "
                     "640x480 demo-scene orbit frames, ground-truth poses; step = integrate + "
                     "raycast of every volume",
         "volumes": 8, "voxels_per_side": 512, "voxel_size_m": 0.004, "image": "640x480",
         "frames": SCHEDULE_DESC,
         "l2": "flushed between timed steps (256 MiB write); volumes 8.6 GB > L2"}
    if n_gpus > 1 and mode == "replicated":
        d["ownership"] = (f"replicated: every rank holds and integrates the 8 volumes and traces every "
                          f"{n_gpus}th 8-pixel block row over all of them; partial maps merged by _hit_wins")
    elif n_gpus > 1:
        d["ownership"] = (f"each 512^3 tile re-tiled into {retile}^3 sub-tiles (2-voxel overlap), "
                          f"sub-tiles owned by {n_gpus} ranks by balanced update counts")
    return d


def peak_hbm() -> tuple[float, str]:
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            return float(json.loads(f.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML clock / throttle-reason sampling every 5 ms in a thread
    (B200_PROFILING.md clocks line); summary over a marked time window."""

    def __init__(self, index: int, period: float = 0.005) -> None:
        self.index, self.period = index, period
        self.samples: list[tuple[float, float, float, int]] = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._nv, self._h = pynvml, h
            self._max = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def _run(self):
        nv, h = self._nv, self._h
        while not self._stop.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                self.samples.append((time.perf_counter(), sm, self._max, rs))
            except Exception:
                pass
            self._stop.wait(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=2)

    def summary(self, t0: float, t1: float) -> dict | None:
        if not self.samples:
            return None
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        rows = inside if len(inside) >= 3 else self.samples
        nv = self._nv
        names = {nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap"}
        active = sorted({n for _, _, _, rs in rows for bit, n in names.items() if rs & bit})
        return {"sm_mhz": statistics.median(r[1] for r in rows), "sm_max_mhz": max(r[2] for r in rows),
                "reasons": active, "samples": len(rows), "samples_in_timed_region": len(inside),
                "window": "timed region" if len(inside) >= 3 else "warm-up + timed region",
                "period_ms": 1e3 * self.period, "source": "NVML"}


def render_frames(poses, intr, scene_fn="demo_scene", max_range=None, procs=None):
    """Depth frames of the synthetic scene (host renderer, identical to the
    reference's), rendered in a process pool; float64 arrays."""
    import multiprocessing as mp
    procs = procs or max(1, min(16, os.cpu_count() or 1))
    mats = [p.matrix for p in poses]
    args = [(m, (intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height), scene_fn, max_range)
            for m in mats]
    if len(args) <= 8 or procs == 1:
        return [_render_one(a) for a in args]
    with mp.get_context("spawn").Pool(procs) as pool:
        return pool.map(_render_one, args, chunksize=max(1, len(args) // (4 * procs)))


def _render_one(a):
    from paper_1511_07106_b200 import geometry, synth
    m, ci, scene_fn, max_range = a
    intr = geometry.CameraIntrinsics(fx=ci[0], fy=ci[1], cx=ci[2], cy=ci[3], width=int(ci[4]),
                                     height=int(ci[5]))
    pose = geometry.Pose(m[:3, :3].copy(), m[:3, 3].copy())
    d = getattr(synth, scene_fn)().render_depth(pose, intr).data
    if max_range is not None:
        d = d.copy()
        d[d > max_range] = 0.0
    return d


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

    from paper_1511_07106_b200 import _native as nat
    from paper_1511_07106_b200.distributed import ShardedFusion, default_retile

    lib = nat.load_library()
    intr, spec, params, poses, scene = workload()
    host_frames = render_frames(poses, intr)
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

    retile = default_retile(world)
    shard = ShardedFusion(spec.keys, spec.voxels_per_side, spec.subvolume_side_length, params,
                          intr, rank, world, retile=retile, mode=os.environ.get("TFB200_SHARD_MODE", "auto"))

    # ---- untimed lap (builds the map) + warm-up ----
    # resident frames have no pending producer (depth_ready=True): each step's
    # culling half runs on the integrator's side stream next to the previous
    # step's raycast, as in the pipeline; at N > 1 the broadcast is the
    # producer (an event after it)
    for i in range(LAP):
        shard.step(dev_frames[i], poses[i], depth_ready=True)
    for i in warm_frames(args.warmup):
        shard.step(dev_frames[i], poses[i], depth_ready=True)
    barrier()

    # ---- timed region: resident inputs, per-step events, L2 flushed between ----
    shard.stats.zero_()
    nat.profile_read()  # drop warm-up records
    lib.tf_profile_enable(1)
    launches0 = lib.tf_launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stops = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    sched = timed_frames(args.steps)
    # at N > 1 every timed step includes the frame's broadcast from rank 0
    # (NCCL over NVLink) into the ranks' frame buffer
    from paper_1511_07106_b200.distributed import broadcast_frame
    frame_buf = torch.empty_like(dev_frames[0])
    with ClockSampler(local) as clocks:
        barrier()
        t0 = time.perf_counter()
        for s, i in enumerate(sched):
            flush.zero_()
            starts[s].record()
            if world > 1:
                if rank == 0:
                    frame_buf.copy_(dev_frames[i])
                broadcast_frame(frame_buf)
                arrived = torch.cuda.Event()
                arrived.record()
                shard.step(frame_buf, poses[i], depth_ready=arrived)
            else:
                shard.step(dev_frames[i], poses[i], depth_ready=True)
            stops[s].record()
        barrier()
        t1 = time.perf_counter()
    lib.tf_profile_enable(0)
    launches = lib.tf_launch_count() - launches0
    shard.check_exchange()
    ms_total = sum(a.elapsed_time(b) for a, b in zip(starts, stops))
    prof = nat.profile_read()
    st = shard.stats.cpu().numpy()
    updates_local = int(st[nat.STAT_VOXEL_UPDATES])
    ms_total = max_over_ranks(ms_total)
    # replicated mode integrates every volume on every rank: count once
    updates = updates_local if shard.replicated else sum_over_ranks(updates_local)
    samples = sum_over_ranks(int(st[nat.STAT_RAY_SAMPLES]))
    ms_per_step = ms_total / args.steps
    fps = 1000.0 / ms_per_step
    updates_per_frame = updates / args.steps
    value = updates_per_frame * fps

    # roofline of the dominant kernel (the voxel-update bracket), this rank
    upd_ms, upd_launches = prof["integrate_update"]
    int_ms, _ = prof["integrate_all"]
    ray_ms, ray_launches = prof["raycast"]
    peak, peak_src = peak_hbm()
    achieved = (BYTES_PER_UPDATE * updates_local / max(upd_launches, 1)) / (
        upd_ms / max(upd_launches, 1) / 1e3) / 1e9 if upd_ms > 0 else 0.0
    traffic = ray_traffic = traffic_src = None
    tfile = ROOT / "profiles" / "traffic_r02d.json"
    if tfile.exists():
        try:
            tj = json.loads(tfile.read_text())
            # the capture is one launch (one frame): its DRAM bytes per update,
            # times this run's updates per launch
            bpu = tj.get("integrate_update_bracket_bytes_per_update")
            traffic = bpu * updates_local / max(upd_launches, 1) if bpu else None
            ray_traffic = tj.get("raycast_bytes_per_launch")
            traffic_src = (f"{tj.get('source')}: {bpu:.2f} DRAM bytes per update x this run's updates per "
                           f"launch" if bpu else tj.get("source"))
        except Exception:
            traffic = ray_traffic = None
    evaluated = samples - sum_over_ranks(int(st[nat.STAT_SUMMARY_SAMPLES]))
    ray_achieved = (64.0 * evaluated / max(ray_launches, 1)) / (ray_ms / max(ray_launches, 1) / 1e3) / 1e9 \
        if ray_ms > 0 else 0.0

    def comp(kind, n_updates):
        ms, n = prof[kind]
        if ms <= 0:
            return None
        gbs = BYTES_PER_UPDATE * n_updates / (ms / 1e3) / 1e9
        return {"ms_per_launch": ms / max(n, 1), "updates_per_launch": n_updates / max(n, 1),
                "achieved_gbs": gbs, "frac": gbs / peak if peak else None}
    free_upd = int(st[nat.STAT_FREE_KERNEL_UPDATES])
    exact_upd = int(st[nat.STAT_EXACT_UPDATES])
    screen_ms, screen_launches = prof["integrate_screen"]
    if prof["integrate_free"][1] == 0:  # free-space bricks inside the streaming kernel (the default)
        components = {
            "brick_apply_kernel (certified free-space bricks + the general bricks' masked updates, one "
            "streaming kernel)": comp("integrate_general", updates_local - exact_upd),
            "exact_queue_kernel (near-surface band, reference arithmetic; beside it on the side stream, "
            "timed only when it runs in stream order)": comp("integrate_exact", exact_upd),
        }
    else:
        components = {
            "brick_free_kernel (certified free-space bricks, bandwidth-bound)": comp("integrate_free", free_upd),
            ("brick_apply_kernel (general bricks: the masked free-space updates)" if screen_launches else
             "brick_update_kernel (general bricks: float32 screen + update in one kernel)"):
                comp("integrate_general", updates_local - free_upd - exact_upd),
            "exact_queue_kernel (near-surface band, reference arithmetic)": comp("integrate_exact", exact_upd),
        }
    # the general bricks' screen runs in the prepare phase (no voxel traffic),
    # on the integrator's side stream next to the previous frame's raycast
    screen = ({"kernel": "brick_update_kernel<true> (float32 screen of the general bricks: masks + exact "
                         "queue; reads the depth tables, not the voxels)",
               "ms_per_launch": screen_ms / screen_launches, "launches": screen_launches,
               "overlaps": "the previous frame's raycast (prepare phase, side stream)",
               "frac_if_serial": (BYTES_PER_UPDATE * updates_local / max(upd_launches, 1)) /
               ((upd_ms + screen_ms) / max(upd_launches, 1) / 1e3) / 1e9 / peak if peak else None}
              if screen_launches else None)

    def per_frame(stat):
        return sum_over_ranks(int(st[stat])) / args.steps

    def per_frame_int(stat):  # integration counters: every rank integrates everything when replicated
        return (int(st[stat]) if shard.replicated else sum_over_ranks(int(st[stat]))) / args.steps

    result = {
        "metric": METRIC, "value": value, "unit": "voxel-updates/s",
        "frames_per_s": fps, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(config_desc(world, retile, shard.mode), **({"raymap_exchange": {
            "p2p": "peer-memory reduce kernel (csrc/comm.cu, CUDA IPC over NVLink)",
            "collective": "NCCL row-block all-to-all + merge + all-gather"}[shard.exchange]}
            if world > 1 else {})),
        "voxel_updates_per_frame": updates_per_frame,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "kernel": "integrate update bracket (brick_apply_kernel: free-space bricks + masked "
                               "updates, with exact_queue_kernel beside it; TF_PROF_INTEGRATE_UPDATE): every "
                               "voxel read/write of the frame's integration", "peak_source": peak_src,
                     "screen": screen,
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
                                  "integrate_screen_overlapped": screen_ms / args.steps,
                                  "integrate_total": int_ms / args.steps,
                                  "raycast": ray_ms / args.steps},
        "integrate": {"noop_updates_per_frame": per_frame_int(nat.STAT_NOOP_UPDATES),
                      "swept_voxels_per_frame": per_frame_int(nat.STAT_SWEPT_VOXELS),
                      "exact_path_voxels_per_frame": per_frame_int(nat.STAT_EXACT_VOXELS),
                      "column_rejected_per_frame": per_frame_int(nat.STAT_COL_SKIPPED),
                      "depth_rejected_per_frame": per_frame_int(nat.STAT_DEPTH_SKIPPED),
                      "active_bricks_per_frame": per_frame_int(nat.STAT_ACTIVE_BRICKS),
                      "free_space_bricks_per_frame": per_frame_int(nat.STAT_FREE_BRICKS),
                      "general_bricks_all_free_per_frame": per_frame_int(nat.STAT_GENERAL_ALL_FREE),
                      "general_parts_all_free_per_frame": per_frame_int(nat.STAT_PART_ALL_FREE),
                      "general_parts_all_skip_per_frame": per_frame_int(nat.STAT_PART_ALL_SKIP),
                      "total_bricks": int(per_frame_int(nat.STAT_TOTAL_BRICKS))},
        "raycast": {"exact_samples_per_frame": per_frame(nat.STAT_EXACT_SAMPLES),
                    "certification_failures": sum_over_ranks(int(st[nat.STAT_CERT_FAILURES])),
                    "summary_certified_samples_per_frame": per_frame(nat.STAT_SUMMARY_SAMPLES),
                    "samples_per_frame": samples / args.steps,
                    "coop_rays_per_frame": per_frame(nat.STAT_COOP_RAYS),
                    "coop_pass_ms_per_frame": prof["raycast_coop"][0] / args.steps,
                    "samples_per_s": samples / (ms_total / 1e3)},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(t0, t1),
    }
    if world > 1:
        result["balance"] = shard.balance_report()

    # ---- e2e through the public pipeline API, frames from pinned host memory ----
    if not args.no_e2e:
        del shard
        torch.cuda.empty_cache()
        result["e2e"] = run_e2e(args, torch, nat, dist, rank, world, intr, spec, params, poses,
                                host_frames, barrier, max_over_ranks, sum_over_ranks)
    else:
        del shard
    del dev_frames
    torch.cuda.empty_cache()

    if world == 1 and not args.no_color:
        result["color"] = run_color(args, torch, spec, params, intr, poses, scene, barrier)
        torch.cuda.empty_cache()
    if world == 1 and not args.no_extra:
        for name, fn in (("config1", run_config1), ("config2", run_config2),
                         ("config4", run_config4), ("config5", run_config5),
                         ("scaling_projection", run_scaling_projection)):
            if args.only and name != args.only:
                continue
            print(f"bench: {name} leg, {torch.cuda.memory_allocated() / 1e9:.1f} GB allocated before",
                  file=sys.stderr, flush=True)
            try:
                result[name] = fn(args, torch, nat, barrier, cpu=not args.no_cpu_baseline)
            except Exception as exc:  # a leg must not take the headline line down
                import traceback
                traceback.print_exc()
                result[name] = {"error": f"{type(exc).__name__}: {exc}"}
            gc.collect()
            torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(intr, spec, params, poses, host_frames)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_color(args, torch, spec, params, intr, poses, scene, barrier) -> dict:
    """Config 3 with an RGB frame fused into a colour channel per volume and
    the model colours rendered every step: device-resident inputs, the same
    frame schedule.  Colour is not in the reference (parity unpinned)."""
    import paper_1511_07106_b200 as tf
    from paper_1511_07106_b200.distributed import ShardedFusion
    from paper_1511_07106_b200.synth import render_rgb

    depth = [torch.from_numpy(scene.render_depth(poses[i], intr).data).cuda() for i in range(LAP)]
    rgb = [torch.from_numpy(render_rgb(scene, poses[i], intr)).cuda() for i in range(LAP)]
    shard = ShardedFusion(spec.keys, spec.voxels_per_side, spec.subvolume_side_length, params, intr,
                          color=True)
    for i in list(range(LAP)) + warm_frames(args.warmup):
        shard.step(depth[i], poses[i], color=rgb[i])
        tf.raycast_colors(shard.tiles, shard.model, poses[i], intr)
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in timed_frames(args.steps):
        shard.step(depth[i], poses[i], color=rgb[i])
        tf.raycast_colors(shard.tiles, shard.model, poses[i], intr)
    b.record()
    barrier()
    ms = a.elapsed_time(b) / args.steps
    del shard
    return {"frames_per_s": 1000.0 / ms, "ms_per_step": ms, "steps": args.steps,
            "path": "ShardedFusion.step(depth, pose, color=rgb) + raycast_colors, inputs resident",
            "note": "colour is not in the reference (parity unpinned); no L2 flush between steps"}


def run_e2e(args, torch, nat, dist, rank, world, intr, spec, params, poses, host_frames,
            barrier, max_over_ranks, sum_over_ranks) -> dict:
    """The headline step through the public FusionPipeline.step API: every
    rank passes its pinned host frame (rank 0's is broadcast when N > 1)."""
    import paper_1511_07106_b200 as tf

    pinned = [torch.from_numpy(f).pin_memory() for f in host_frames]
    cfg = tf.RunConfig(side_length=4.08, resolution=1020, resident_resolution=510,
                       use_groundtruth=True, max_resident=8)
    spill = tempfile.mkdtemp(prefix="tfb200_spill_")
    pipe = tf.FusionPipeline(cfg, spill, rank=rank, world=world)
    result = torch.empty(pipe.stats.shape, dtype=pipe.stats.dtype).pin_memory()

    def step(i):
        pipe.step(pinned[i], poses[i])               # public API: H2D inside step()
        result.copy_(pipe.stats, non_blocking=True)  # D2H of the step's counters
        return result

    for i in list(range(LAP)) + warm_frames(args.warmup):
        out = step(i)
    torch.cuda.synchronize()
    barrier()
    before = int(out[nat.STAT_VOXEL_UPDATES])
    # every step uploads its frame from pinned memory and reads its counters
    # back into pinned memory, both stream-ordered; the host waits once at
    # the end (the last read has landed when the clock stops)
    t0 = time.perf_counter()
    for i in timed_frames(args.steps):
        out = step(i)
    torch.cuda.synchronize()
    barrier()
    sec = max_over_ranks(time.perf_counter() - t0)
    upd = int(out[nat.STAT_VOXEL_UPDATES]) - before
    updates = upd if (pipe._shard is not None and pipe._shard.replicated) else sum_over_ranks(upd)
    del pipe
    return {"value": updates / sec, "unit": "voxel-updates/s", "frames_per_s": args.steps / sec,
            "h2d_bytes_per_step": int(host_frames[0].nbytes) if rank == 0 else 0,
            "d2h_bytes_per_step": int(out.numel() * out.element_size()), "steps": args.steps,
            "path": "FusionPipeline.step(pinned host frame)" +
                    (f" at world {world} (rank-0 H2D + broadcast)" if world > 1 else "")}


# ---------------------------------------------------------------------------
# extra legs (N = 1): the other BASELINE configs
# ---------------------------------------------------------------------------

def _pipeline_run(torch, pipe, frames_pinned, poses, first_gt=True):
    """Frames through FusionPipeline.step (pinned host frames), host waits
    once at the end; returns seconds."""
    t0 = time.perf_counter()
    for i, f in enumerate(frames_pinned):
        pipe.step(f, poses[i])
    torch.cuda.synchronize()
    return time.perf_counter() - t0


def run_config1(args, torch, nat, barrier, cpu: bool) -> dict:
    """BASELINE configs[0]: one 256^3 volume (init_grid(3.0, 254, 254)), 64
    orbit frames, ground-truth poses, through FusionPipeline.step from pinned
    host frames; frames/s excludes frame 0 (evaluation.py:112-119).  CPU: the
    oracle over the same 64 frames on all host threads."""
    import paper_1511_07106_b200 as tf

    cfg = tf.RunConfig(side_length=3.0, resolution=254, resident_resolution=254,
                       use_groundtruth=True)
    intr = cfg.intrinsics()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, LAP)
    host = render_frames(poses, intr)
    pinned = [torch.from_numpy(f).pin_memory() for f in host]
    warm = tf.FusionPipeline(cfg, tempfile.mkdtemp(prefix="tfb200_c1w_"))
    _pipeline_run(torch, warm, pinned, poses)
    del warm
    pipe = tf.FusionPipeline(cfg, tempfile.mkdtemp(prefix="tfb200_c1_"))
    pipe.step(pinned[0], poses[0])
    torch.cuda.synchronize()
    pipe.stats.zero_()
    gc.disable()
    sec = _pipeline_run(torch, pipe, pinned[1:], poses[1:])
    gc.enable()
    ks = pipe.kernel_stats()
    out = {"workload": "configs[0]: one 256^3 volume (init_grid(3.0, 254, 254)), 640x480, 64 orbit "
                       "frames, ground-truth poses, FusionPipeline.step from pinned host frames",
           "frames": LAP - 1, "frames_per_s": (LAP - 1) / sec,
           "voxel_updates_per_s": ks["voxel_updates"] / sec,
           "voxel_updates_per_frame": ks["voxel_updates"] / (LAP - 1)}
    if cpu:
        import oracle
        spec = tf.init_grid(3.0, 254, 254)
        params = tf.FusionParams.for_voxel_size(spec.voxel_size)
        out["cpu"] = _cpu_static(oracle, spec, params, intr, poses, host, list(range(1, LAP)),
                                 warm=[0], kind="full 64-frame run (frame 0 untimed)")
    return out


def run_config2(args, torch, nat, barrier, cpu: bool) -> dict:
    """BASELINE configs[1]: one 256^3 volume, ICP tracking on, 1.5-degree orbit
    (64 frames).  CPU: the oracle's integrate / raycast / track on all host
    threads over the first 9 frames (8 tracked), per frame."""
    import paper_1511_07106_b200 as tf

    cfg = tf.RunConfig(side_length=3.0, resolution=254, resident_resolution=254,
                       use_groundtruth=False)
    intr = cfg.intrinsics()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, 240)[:LAP]
    host = render_frames(poses, intr)
    frames = [torch.from_numpy(f).cuda() for f in host]
    warm = tf.FusionPipeline(cfg, tempfile.mkdtemp(prefix="tfb200_c2w_"))
    for i, f in enumerate(frames):
        warm.step(f, poses[i] if i == 0 else None)
    torch.cuda.synchronize()
    del warm
    pipe = tf.FusionPipeline(cfg, tempfile.mkdtemp(prefix="tfb200_c2_"))
    pipe.step(frames[0], poses[0])   # frame 0 defines the world frame
    gc.collect()
    barrier()
    pipe.stats.zero_()
    gc.disable()  # no collector pause inside the short timed pass
    t0 = time.perf_counter()
    for i in range(1, LAP):
        pipe.step(frames[i])
    barrier()
    sec = time.perf_counter() - t0
    gc.enable()
    ks = pipe.kernel_stats()
    lost = sum(1 for r in pipe.records[1:] if not r.tracked)
    err = max(float(np.abs(p.translation - q.translation).max()) for p, q in zip(pipe.poses, poses))
    out = {"workload": "configs[1]: one 256^3 volume (init_grid(3.0, 254, 254)), 640x480, "
                       "1.5-degree orbit, ICP tracking on (frames resident)", "frames": LAP - 1,
           "frames_per_s": (LAP - 1) / sec, "voxel_updates_per_s": ks["voxel_updates"] / sec,
           "lost_frames": lost, "max_translation_error_m": err}
    if cpu:
        import oracle
        spec = tf.init_grid(3.0, 254, 254)
        params = tf.FusionParams.for_voxel_size(spec.voxel_size)
        out["cpu"] = _cpu_tracked(oracle, spec, params, intr, poses, host, 9)
    return out


CONFIG4 = dict(frames=2000, length=20.0, block_voxels=258, block_side_length=1.024,
               max_volumes=16, hysteresis=1.5, max_range=4.0)


def run_config4(args, torch, nat, barrier, cpu: bool) -> dict:
    """BASELINE configs[3]: dynamic placement over the 2000-frame corridor
    (synth.corridor_scene, corridor_trajectory(20, 2000), depth > 4 m zeroed,
    258^3 tiles at 4 mm, at most 16 tiles, hysteresis 1.5, ground-truth poses),
    every frame through FusionPipeline.step from pinned host frames: placement
    (device endpoint histogram + host update_allocation), integration and
    raycast of the allocated tiles, removal (extraction of retired tiles)."""
    import paper_1511_07106_b200 as tf

    c = CONFIG4
    cfg = tf.RunConfig(dynamic=True, block_voxels=c["block_voxels"],
                       block_side_length=c["block_side_length"], max_volumes=c["max_volumes"],
                       hysteresis=c["hysteresis"], max_resident=c["max_volumes"], use_groundtruth=True)
    intr = cfg.intrinsics()
    poses = tf.corridor_trajectory(c["length"], c["frames"])
    t_r = time.perf_counter()
    host = render_frames(poses, intr, "corridor_scene", c["max_range"])
    render_s = time.perf_counter() - t_r
    pinned = [torch.from_numpy(f).pin_memory() for f in host]
    warm = tf.FusionPipeline(cfg, tempfile.mkdtemp(prefix="tfb200_c4w_"))
    _pipeline_run(torch, warm, pinned[:50], poses[:50])
    del warm
    torch.cuda.empty_cache()
    pipe = tf.FusionPipeline(cfg, tempfile.mkdtemp(prefix="tfb200_c4_"))
    pipe.step(pinned[0], poses[0])
    torch.cuda.synchronize()
    pipe.stats.zero_()
    gc.disable()
    sec = _pipeline_run(torch, pipe, pinned[1:], poses[1:])
    gc.enable()
    ks = pipe.kernel_stats()
    n = c["frames"] - 1
    vols = [r.volumes for r in pipe.records]
    out = {"workload": "configs[3]: dynamic placement, corridor_trajectory(20.0, 2000), 640x480, "
                       "258^3 tiles at 4 mm, max_volumes 16, hysteresis 1.5, depth > 4 m zeroed, "
                       "ground-truth poses, pinned host frames", "frames": n,
           "frames_per_s": n / sec, "voxel_updates_per_s": ks["voxel_updates"] / sec,
           "voxel_updates_per_frame": ks["voxel_updates"] / n, "max_live_tiles": max(vols),
           "distinct_tiles": len(set(k for k in pipe.volumes.keys())) + len(pipe._archive),
           "host_render_s": render_s}
    if cpu:
        import oracle
        out["cpu"] = _cpu_dynamic(oracle, cfg, intr, poses, host, 50)
    del pipe
    return out


def run_config5(args, torch, nat, barrier, cpu: bool) -> dict:
    """BASELINE configs[4], one GPU's share: 4 of the 32 1024^3 tiles (~1 mm
    voxels; the 4x4x2 key block, spacing 1022) — the 4 rank 0 owns at N = 8 —
    with max_resident = 2, so every frame evicts tiles to the pinned-host
    spill tier (async D2H/H2D side stream) and brings others back.  Run with
    the exact tier ("host", 8 B/voxel) and the opt-in packed capacity mode
    ("host_packed", half tsdf + uint8 weight, 3 B/voxel); reports frames/s,
    spill GB/s, the pinned copy bandwidth measured alongside, and the packed
    run's tsdf error against the exact run (weights must agree)."""
    import psutil

    import paper_1511_07106_b200 as tf
    from paper_1511_07106_b200.distributed import owned_keys
    from paper_1511_07106_b200.volumes import VolumeSet

    n = 1024
    tile_bytes = n ** 3 * 8
    if psutil.virtual_memory().available < 6 * tile_bytes:
        return {"skipped": f"needs ~{6 * tile_bytes / 1e9:.0f} GB free host memory for the spill tier"}
    vs = 0.001
    keys = [(x * 1022, y * 1022, z * 1022) for x in (-2, -1, 0, 1) for y in (-2, -1, 0, 1)
            for z in (0, 1)]
    mine = owned_keys(keys, 0, 8)
    params = tf.FusionParams.for_voxel_size(vs)
    intr = tf.RunConfig().intrinsics()
    poses = tf.orbit_trajectory((0.0, 0.0, 1.5), 1.5, LAP)
    frame_ids = [0, 16, 32, 48]
    host = render_frames([poses[i] for i in frame_ids], intr)
    pinned = [torch.from_numpy(f).pin_memory() for f in host]
    # pinned copy bandwidth on this box, for the spill rate's denominator
    src = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    dst = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
    t0 = time.perf_counter()
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    d2h = (1 << 30) / (time.perf_counter() - t0) / 1e9
    t0 = time.perf_counter()
    src.copy_(dst, non_blocking=True)
    torch.cuda.synchronize()
    h2d = (1 << 30) / (time.perf_counter() - t0) / 1e9
    del src, dst
    stats = nat.stats.buffer()

    def run(tier):
        vset = VolumeSet(params, voxels_per_side=n, voxel_size=vs, max_resident=2,
                         spill_dir=tempfile.mkdtemp(prefix="tfb200_c5_"), spill_tier=tier)
        for k in mine:
            vset.add(k)

        def frame(j):
            depth = torch.empty(host[j].shape, dtype=torch.float64, device="cuda")
            depth.copy_(pinned[j], non_blocking=True)
            rm = tf.RayMap.empty(intr)
            for k in vset.keys():
                tile = vset.acquire(k)
                tf.integrate_volumes([tile], depth, poses[frame_ids[j]], intr, params, stats)
                tf.raycast_volumes([tile], poses[frame_ids[j]], intr, rm, params, stats)
                vset.release(k)
            return rm

        counts = []
        frame(0)
        counts.append((vset.files_read, vset.files_written))
        torch.cuda.synchronize()
        print(f"bench: config5 {tier}: {torch.cuda.memory_allocated() / 1e9:.1f} GB allocated after frame 0",
              file=sys.stderr, flush=True)
        stats.zero_()
        b0 = (vset.link_bytes_read, vset.link_bytes_written)
        t0 = time.perf_counter()
        for j in range(1, len(frame_ids)):
            frame(j)
            counts.append((vset.files_read, vset.files_written))
        torch.cuda.synchronize()
        sec = time.perf_counter() - t0
        moved = (vset.link_bytes_read - b0[0]) + (vset.link_bytes_written - b0[1])
        nf = len(frame_ids) - 1
        return vset, {"frames_per_s": nf / sec,
                      "voxel_updates_per_s": int(stats[nat.STAT_VOXEL_UPDATES].item()) / sec,
                      "link_bytes_per_frame": moved / nf, "link_gbs": moved / sec / 1e9}, counts

    exact_set, exact, schedule = run("host")
    packed_set, packed, _ = run("host_packed")
    ref_schedule = reference_spill_schedule(mine, len(frame_ids))
    tau = params.truncation
    err, wdiff = 0.0, 0
    for k in exact_set.keys():  # tile by tile, both resident at once
        a = exact_set.acquire(k)
        b = packed_set.acquire(k)
        err = max(err, float((a.voxels[..., 0] - b.voxels[..., 0]).abs().max().item()))
        wdiff += int((a.voxels[..., 1] != b.voxels[..., 1]).sum().item())
        exact_set.release(k)
        packed_set.release(k)
    packed.update({"max_tsdf_error_over_tau": err / tau, "weight_mismatches": wdiff,
                   "note": "opt-in capacity mode, not the parity format"})
    del exact_set, packed_set
    nf = len(frame_ids) - 1
    return {"workload": "configs[4], one GPU's share at N = 8: 4 tiles of 1024^3 at 1 mm (4x4x2 key "
                        "block, spacing 1022; rank 0's of 8), max_resident 2 -> pinned-host spill "
                        "every frame; orbit frames 16, 32, 48 timed (0 untimed)",
            "tiles": len(mine), "tile_bytes": tile_bytes, "frames": nf,
            "frames_per_s": exact["frames_per_s"], "voxel_updates_per_s": exact["voxel_updates_per_s"],
            "spill_bytes_per_frame": exact["link_bytes_per_frame"], "spill_gbs": exact["link_gbs"],
            "pinned_d2h_gbs": d2h, "pinned_h2d_gbs": h2d, "packed_tier": packed,
            "spill_schedule": {"files_read_written_after_each_frame": schedule,
                               "reference": ref_schedule,
                               "matches_reference": ref_schedule is None or ref_schedule == schedule,
                               "how": "the unmodified reference VolumeSet (baseline/_ref) driven through the "
                                      "same acquire / release sequence on 8^3 stand-in tiles"},
            "bound": "host link (each frame moves every tile through the spill tier)"}


def run_scaling_projection(args, torch, nat, barrier, cpu: bool) -> dict:
    """A projection, not a measurement (this pool has one GPU): config 3
    re-tiled and owned as N ranks would own it (distributed.retile,
    balanced_owners on the work the culling stage measured over the lap),
    then every timed frame runs each rank's share — integrate + raycast of its
    sub-tiles into a partial map — one rank after the other on this GPU, with
    CUDA events around each.  The frame's projected time is the slowest
    rank's; the ray-map reduction (peer memory over NVLink, ~9 MB per rank per
    frame) and the frame broadcast are not included."""
    import paper_1511_07106_b200 as tf
    from paper_1511_07106_b200.distributed import balanced_owners, default_retile, retile

    intr, spec, params, poses, scene = workload()
    host = render_frames(poses, intr)
    frames = [torch.from_numpy(f).cuda() for f in host]
    out = {"note": "projection from one GPU: per-rank shares timed one after the other; the exchange "
                   "and the broadcast are not included; the driver's SCALE run measures the real thing"}
    # replicated mode (ShardedFusion's default when the map fits): every rank
    # integrates all 8 volumes and traces every n-th block row over them
    tiles = [tf.TsdfSubvolume.empty(k, spec.voxels_per_side, spec.subvolume_side_length) for k in spec.keys]
    for i in range(LAP):
        tf.integrate_volumes(tiles, frames[i], poses[i], intr, params)
    torch.cuda.synchronize()
    rep = {n: [] for n in (2, 4, 8)}
    for i in timed_frames(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        tf.integrate_volumes(tiles, frames[i], poses[i], intr, params)
        b.record()
        ev = []
        for n in (2, 4, 8):
            for r in range(n):
                c, d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                rm = tf.RayMap.empty(intr)
                c.record()
                tf.raycast_volumes(tiles, poses[i], intr, rm, params, rows=(r, n))
                d.record()
                ev.append((n, r, c, d))
        torch.cuda.synchronize()
        t_int = a.elapsed_time(b)
        for n in (2, 4, 8):
            rep[n].append(t_int + max(c.elapsed_time(d) for m, r, c, d in ev if m == n))
    for n in (2, 4, 8):
        mean = sum(rep[n]) / len(rep[n])
        out[f"replicated_n{n}"] = {"projected_ms_per_frame": mean, "projected_frames_per_s": 1000.0 / mean}
    del tiles
    torch.cuda.empty_cache()
    for n in (2, 4, 8):
        k = default_retile(n, spec.voxels_per_side)
        units, m = retile(spec.keys, spec.voxels_per_side, spec.voxel_size, k)
        counters = torch.zeros((len(units), 2), dtype=torch.int64, device="cuda")
        tiles = []
        for u, key in enumerate(units):
            t = tf.TsdfSubvolume.empty(key, m, m * spec.voxel_size)
            t.counters = counters[u]
            tiles.append(t)
        for i in range(LAP):
            tf.integrate_volumes(tiles, frames[i], poses[i], intr, params)
        c = counters.to(torch.float64)
        costs = (c[:, 0] * 4.0 + c[:, 1]).cpu().tolist()
        owners = balanced_owners(costs, n)
        shares = [[tiles[u] for u in range(len(units)) if owners[u] == r] for r in range(n)]
        for i in warm_frames(args.warmup):  # untimed: each share's first raycast sizes its scratch
            for r in range(n):
                tf.integrate_volumes(shares[r], frames[i], poses[i], intr, params)
                tf.raycast_volumes(shares[r], poses[i], intr, tf.RayMap.empty(intr), params)
        torch.cuda.synchronize()
        per_frame = []
        per_rank = [0.0] * n
        for i in timed_frames(args.steps):
            times = []
            for r in range(n):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                rm = tf.RayMap.empty(intr)
                a.record()
                tf.integrate_volumes(shares[r], frames[i], poses[i], intr, params)
                tf.raycast_volumes(shares[r], poses[i], intr, rm, params)
                b.record()
                times.append((a, b))
            torch.cuda.synchronize()
            ms = [a.elapsed_time(b) for a, b in times]
            per_frame.append(max(ms))
            for r in range(n):
                per_rank[r] += ms[r] / len(timed_frames(args.steps))
        mean = sum(per_frame) / len(per_frame)
        out[f"volumes_n{n}"] = {"retile": k, "sub_tiles": len(units), "sub_tile_voxels": m,
                        "projected_ms_per_frame": mean, "projected_frames_per_s": 1000.0 / mean,
                        "per_rank_ms": per_rank,
                        "imbalance_max_over_mean": max(per_rank) / (sum(per_rank) / n)}
        del tiles, shares, counters
        torch.cuda.empty_cache()
    return out


def reference_spill_schedule(keys, nframes):
    """(files_read, files_written) after each frame from the reference's own
    VolumeSet (volumes.py:156-302) for config 5's acquire / release order, on
    tiny stand-in tiles (the counts do not depend on the tile size); None when
    baseline/_ref is absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "tilefusion").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="tfb200_numba_"))
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import tilefusion as rtf
    vs = 0.001
    rset = rtf.VolumeSet(rtf.FusionParams.for_voxel_size(vs), voxels_per_side=8, voxel_size=vs,
                         max_resident=2, spill_dir=tempfile.mkdtemp(prefix="tfb200_refspill_"))
    for k in keys:
        rset.add(k)
    out = []
    for _ in range(nframes):
        for k in rset.keys():
            rset.acquire(k)
            rset.release(k)
        out.append((rset.files_read, rset.files_written))
    return out


# ---------------------------------------------------------------------------
# CPU baselines (oracle restatement of the reference kernels, all host threads)
# ---------------------------------------------------------------------------

def _coarse(params, vs):
    return max(2, int(round(0.5 * params.truncation / vs)))


def _oracle_frame(oracle, tiles, keys, vs, params, intr, pose, depth, threads, raycast=True):
    inv = pose.invert()
    t0 = time.perf_counter()
    updates = 0
    for (t, w), k in zip(tiles, keys):
        updates += oracle.integrate(t, w, k, vs, depth, inv.rotation, inv.translation,
                                    pose.translation, intr.fx, intr.fy, intr.cx, intr.cy,
                                    params.truncation, params.max_weight, params.sample_weight,
                                    threads=threads)
    t_int = time.perf_counter() - t0
    maps = None
    t_ray = 0.0
    if raycast:
        d = np.full((intr.height, intr.width), np.inf)
        v = np.zeros((intr.height, intr.width, 3))
        nn = np.zeros_like(v)
        t0 = time.perf_counter()
        for (t, w), k in zip(tiles, keys):
            oracle.raycast(t, w, k, vs, params.truncation, _coarse(params, vs), pose.rotation,
                           pose.translation, intr.fx, intr.fy, intr.cx, intr.cy, d, v, nn,
                           threads=threads)
        t_ray = time.perf_counter() - t0
        maps = (d, v, nn)
    return updates, t_int, t_ray, maps


def _cpu_static(oracle, spec, params, intr, poses, frames, timed, warm=(), kind=""):
    threads = oracle.default_threads()
    n = spec.voxels_per_side
    tiles = [(np.zeros((n, n, n), np.float32), np.zeros((n, n, n), np.float32)) for _ in spec.keys]
    for i in warm:
        _oracle_frame(oracle, tiles, spec.keys, spec.voxel_size, params, intr, poses[i], frames[i],
                      threads, raycast=False)
    tot, ups = 0.0, 0
    for i in timed:
        u, ti, tr, _ = _oracle_frame(oracle, tiles, spec.keys, spec.voxel_size, params, intr, poses[i],
                                     frames[i], threads)
        tot += ti + tr
        ups += u
    return {"frames_per_s": len(timed) / tot, "voxel_updates_per_s": ups / tot, "cores": threads,
            "kind": "port", "sample": kind}


def _cpu_tracked(oracle, spec, params, intr, poses, frames, nframes):
    """Config 2 on the CPU: per frame oracle.track against the previous model,
    then integrate + raycast at the tracked pose (pipeline.py:117-172)."""
    import paper_1511_07106_b200 as tf
    threads = oracle.default_threads()
    n = spec.voxels_per_side
    vs = spec.voxel_size
    tiles = [(np.zeros((n, n, n), np.float32), np.zeros((n, n, n), np.float32)) for _ in spec.keys]
    pose = poses[0]
    _, _, _, model = _oracle_frame(oracle, tiles, spec.keys, vs, params, intr, pose, frames[0], threads)
    tot, t_track, lost = 0.0, 0.0, 0
    for i in range(1, nframes):
        t0 = time.perf_counter()
        rot, t, is_lost, _, _ = oracle.track(frames[i], intr.fx, intr.fy, intr.cx, intr.cy, *model,
                                             pose.rotation, pose.translation, pose.rotation,
                                             pose.translation)
        dt = time.perf_counter() - t0
        t_track += dt
        if is_lost:
            lost += 1
        else:
            pose = tf.Pose(rot, t)
        _, ti, tr, model = _oracle_frame(oracle, tiles, spec.keys, vs, params, intr, pose, frames[i],
                                         threads)
        tot += dt + ti + tr
    k = nframes - 1
    return {"frames_per_s": k / tot, "track_s_per_frame": t_track / k, "lost_frames": lost,
            "cores": threads, "kind": "port",
            "sample": f"frames 1-{k} of the run (frame 0 untimed): oracle.track + integrate + raycast"}


def _cpu_dynamic(oracle, cfg, intr, poses, frames, nframes):
    """Config 4's first frames on the CPU: placement (oracle endpoint cells +
    the reference's histogram and update_allocation), then integrate + raycast
    of every allocated tile (tiles retired by placement are dropped; the
    extraction of retired tiles is not timed here)."""
    from paper_1511_07106_b200.volumes import AllocationPolicy, update_allocation
    threads = oracle.default_threads()
    spacing = cfg.block_voxels - 2
    vs = cfg.block_side_length / spacing
    n = cfg.block_voxels
    params = cfg.fusion_params(vs)
    policy = AllocationPolicy(max_volumes=cfg.max_volumes, hysteresis=cfg.hysteresis)
    tiles: dict = {}
    tot, ups = 0.0, 0
    for i in range(nframes):
        t0 = time.perf_counter()
        p = poses[i]
        counts = oracle.bin_endpoints(frames[i], intr.fx, intr.fy, intr.cx, intr.cy, p.rotation,
                                      p.translation, spacing, vs)
        added, removed = update_allocation(tuple(tiles), counts, policy)
        for k in removed:
            del tiles[k]
        for k in added:
            tiles[k] = (np.zeros((n, n, n), np.float32), np.zeros((n, n, n), np.float32))
        dt = time.perf_counter() - t0
        u, ti, tr, _ = _oracle_frame(oracle, list(tiles.values()), list(tiles), vs, params, intr, p,
                                     frames[i], threads)
        if i > 0:
            tot += dt + ti + tr
            ups += u
    k = nframes - 1
    return {"frames_per_s": k / tot, "voxel_updates_per_s": ups / tot, "cores": threads,
            "kind": "port", "sample": f"frames 1-{k} of the 2000 (frame 0 untimed)"}


class OracleMap:
    """The config-3 map on the host (oracle arrays), advanced through the same
    frame schedule as the GPU arm."""

    def __init__(self, oracle, intr, spec, params, poses, frames, threads):
        self.o, self.intr, self.spec, self.params = oracle, intr, spec, params
        self.poses, self.frames, self.threads = poses, frames, threads
        n = spec.voxels_per_side
        self.tiles = [(np.zeros((n, n, n), np.float32), np.zeros((n, n, n), np.float32))
                      for _ in spec.keys]

    def integrate_only(self, i):
        _oracle_frame(self.o, self.tiles, self.spec.keys, self.spec.voxel_size, self.params,
                      self.intr, self.poses[i], self.frames[i], self.threads, raycast=False)

    def step(self, i, subset=None):
        """integrate every tile (the map state must follow the GPU arm's),
        raycast the tiles in ``subset``; returns (updates, integrate s, raycast s
        scaled to all tiles)."""
        ups, ti, _, _ = _oracle_frame(self.o, self.tiles, self.spec.keys, self.spec.voxel_size,
                                      self.params, self.intr, self.poses[i], self.frames[i],
                                      self.threads, raycast=False)
        idx = list(range(len(self.tiles))) if subset is None else subset
        _, _, tr, _ = _oracle_frame(self.o, [self.tiles[j] for j in idx],
                                    [self.spec.keys[j] for j in idx], self.spec.voxel_size,
                                    self.params, self.intr, self.poses[i], self.frames[i],
                                    self.threads)
        return ups, ti, tr * len(self.tiles) / len(idx)


def cpu_baseline(intr, spec, params, poses, host_frames) -> dict:
    """The oracle on all host threads on a bounded sample of the same workload:
    the lap that builds the map, then 3 frames of the timed schedule."""
    import oracle

    threads = oracle.default_threads()
    m = OracleMap(oracle, intr, spec, params, poses, host_frames, threads)
    t0 = time.perf_counter()
    for i in range(LAP):
        m.integrate_only(i)
    lap_s = time.perf_counter() - t0
    times, ups = [], []
    for i in timed_frames(3):
        u, ti, tr = m.step(i)
        times.append(ti + tr)
        ups.append(u)
    frame_s = sum(times) / len(times)
    return {"value": sum(ups) / sum(times), "unit": "voxel-updates/s", "cores": threads, "kind": "port",
            "frames_per_s": 1.0 / frame_s,
            "sample": f"the map after the 64-frame lap (integrated untimed, {lap_s:.0f} s), then 3 "
                      f"frames of the timed schedule (integrate + raycast of all 8 volumes), C oracle "
                      f"on {threads} host threads"}


def numba_sample(intr, spec, params, poses, host_frames, m: OracleMap, frame: int, tiles: list) -> dict:
    """The unmodified reference package (baseline/_ref, numba, single core)
    on a bounded sample: its public integrate + raycast on ``tiles`` of the
    map state ``m`` holds (copied), frame ``frame``; scaled to 8 tiles."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "tilefusion").exists():
        return {"unavailable": "baseline/_ref not installed"}
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="tfb200_numba_"))
    sys.path.insert(0, str(ref))
    import tilefusion as rtf

    rintr = rtf.CameraIntrinsics(fx=intr.fx, fy=intr.fy, cx=intr.cx, cy=intr.cy, width=intr.width,
                                 height=intr.height)
    rparams = rtf.FusionParams.for_voxel_size(spec.voxel_size)
    # JIT warm-up on a tiny volume (compilation excluded)
    small = rtf.TsdfSubvolume.empty(np.array([-8, -8, 100]), 16, 16 * spec.voxel_size)
    f0 = rtf.DepthFrame(host_frames[frame])
    p = poses[frame]
    rpose = rtf.Pose(p.rotation.copy(), p.translation.copy())
    rtf.integrate(small, f0, rpose, rintr, rparams)
    rtf.raycast(small, rpose, rintr, rtf.RayMap.empty(rintr), rparams)
    t_int = t_ray = 0.0
    rm = rtf.RayMap.empty(rintr)
    for j in tiles:
        vol = rtf.TsdfSubvolume.empty(np.array(spec.keys[j]), spec.voxels_per_side,
                                      spec.subvolume_side_length)
        np.copyto(vol.tsdf, m.tiles[j][0])
        np.copyto(vol.weight, m.tiles[j][1])
        t0 = time.perf_counter()
        rtf.integrate(vol, f0, rpose, rintr, rparams)
        t_int += time.perf_counter() - t0
        t0 = time.perf_counter()
        rtf.raycast(vol, rpose, rintr, rm, rparams)
        t_ray += time.perf_counter() - t0
        del vol
    scale = len(spec.keys) / len(tiles)
    frame_s = (t_int + t_ray) * scale
    return {"frames_per_s": 1.0 / frame_s, "integrate_s_per_volume": t_int / len(tiles),
            "raycast_s_per_volume": t_ray / len(tiles), "cores": 1, "kind": "reference",
            "sample": f"unmodified reference (baseline/_ref, numba, single core): tilefusion.integrate + "
                      f"tilefusion.raycast of frame {frame} into tiles {tiles} of the same map state "
                      f"(copied from the oracle arm), scaled to 8 tiles; JIT excluded"}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # the CPU reference runs once, on rank 0
    import oracle

    world = int(os.environ.get("WORLD_SIZE", "1"))
    threads = oracle.default_threads()
    intr, spec, params, poses, scene = workload()
    host_frames = render_frames(poses, intr)
    m = OracleMap(oracle, intr, spec, params, poses, host_frames, threads)
    t0 = time.perf_counter()
    for i in range(LAP):
        m.integrate_only(i)
    lap_s = time.perf_counter() - t0
    steps, warmup = max(1, args.steps), max(0, args.warmup)
    # every step integrates all 8 tiles (the map follows the GPU arm's); the
    # raycast is timed on a round-robin subset when K is large, scaled to 8
    per = max(1, min(8, 512 // steps))
    for i in warm_frames(warmup):
        m.integrate_only(i)
    times, ups = [], []
    for s, i in enumerate(timed_frames(steps)):
        subset = [(s * per + j) % 8 for j in range(per)]
        u, ti, tr = m.step(i, subset)
        times.append(ti + tr)
        ups.append(u)
    frame_s = sum(times) / len(times)
    value = sum(ups) / sum(times)
    sample = (f"per step: the GPU arm's frame on the same map state (64-frame lap + warm-up "
              f"frames integrated untimed first, {lap_s:.0f} s); integrate of all 8 volumes + raycast "
              f"of {per} of 8 (round-robin, scaled to 8); C restatement of the reference kernels on "
              f"{threads} host threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "voxel-updates/s",
        "frames_per_s": 1.0 / frame_s, "n_gpus": world, "steps": steps, "warmup": warmup,
        "ms_per_step": frame_s * 1e3, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_desc(1),
        "cpu_baseline": {"value": value, "unit": "voxel-updates/s", "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "voxel-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}
    if not args.no_numba:
        try:
            nb = numba_sample(intr, spec, params, poses, host_frames, m, timed_frames(steps)[-1],
                              [2, 6])
        except Exception as exc:
            nb = {"error": f"{type(exc).__name__}: {exc}"}
        line["cpu_baseline_reference_numba"] = nb
    print(json.dumps(line), flush=True)


def main() -> None:
    args = parse_args()
    relaunch_if_needed(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
