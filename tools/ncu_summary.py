"""Key metrics per kernel from an `ncu --set full` report (developer tool):

    python tools/ncu_summary.py report.ncu-rep > summary.txt
    python tools/ncu_summary.py report.ncu-rep --traffic traffic.json

Per launch: duration, DRAM bytes, registers, occupancy, warps/issue active,
local and global request counts, global sectors per request, and the stall
breakdown from the source-level samples.  --traffic writes the update
bracket's and the raycast's DRAM bytes per launch for bench.py.
"""
import csv
import io
import json
import subprocess
import sys

M = [("gpu__time_duration.sum", "duration_us"), ("dram__bytes_read.sum", "dram_read"),
     ("dram__bytes_write.sum", "dram_write"), ("launch__registers_per_thread", "registers"),
     ("launch__occupancy_limit_registers", "occ_limit_regs_blocks"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
     ("smsp__inst_executed.sum", "warp_instructions"),
     ("l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum", "local_ld_requests"),
     ("l1tex__t_requests_pipe_lsu_mem_local_op_st.sum", "local_st_requests"),
     ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global_ld_requests"),
     ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global_ld_sectors"),
     ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
     ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct")]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m, name in M:
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                try:
                    d[name] = float(v)
                except ValueError:
                    d[name] = v
                if name == "duration_us":
                    d[name] *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
                                "second": 1e6}.get(units[hdr.index(m)], 1.0)
                if name.startswith("dram") and units[hdr.index(m)] == "Mbyte":
                    d[name] *= 1e6
                if name.startswith("dram") and units[hdr.index(m)] == "Kbyte":
                    d[name] *= 1e3
                if name.startswith("dram") and units[hdr.index(m)] == "Gbyte":
                    d[name] *= 1e9
        res.append(d)
    return res


def stalls(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kernel}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    hdr = rows[1]
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    agg = {}
    for r in rows[2:]:
        if len(r) != len(hdr) or not r[0].startswith("0x"):
            continue
        for i in cols:
            try:
                agg[hdr[i]] = agg.get(hdr[i], 0.0) + float(r[i] or 0)
            except ValueError:
                pass
    tot = sum(agg.values()) or 1.0
    return {k[6:]: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:6]}


def main():
    rep = sys.argv[1]
    rs = raw(rep)
    if "--traffic" in sys.argv:
        out = sys.argv[sys.argv.index("--traffic") + 1]
        by = {}
        for d in rs:
            by.setdefault(d["kernel"], []).append(d.get("dram_read", 0) + d.get("dram_write", 0))
        avg = {k: sum(v) / len(v) for k, v in by.items()}
        def short(k):
            return k.split("::")[-1].replace("void ", "")

        def screen(k):  # the prepare-phase screen (no voxel traffic; not in the bracket)
            return any(f"brick_update_kernel<{t}>" in short(k) for t in ("true", "(bool)1", "1"))

        bracket = sum(v for k, v in avg.items()
                      if short(k).split("<")[0] in ("brick_update_kernel", "brick_apply_kernel",
                                                    "brick_free_kernel", "exact_queue_kernel") and not screen(k))
        ray = next((v for k, v in avg.items() if "raycast_kernel" in k), None)
        scr = next((v for k, v in avg.items() if screen(k)), None)
        frame_updates = float(sys.argv[sys.argv.index("--updates") + 1]) if "--updates" in sys.argv else None
        json.dump({"source": f"ncu --set full capture {rep.split('/')[-1]}, one timed-region launch per kernel "
                             "(frame 0 of the orbit)",
                   "integrate_update_bracket_bytes_per_launch": bracket, "raycast_bytes_per_launch": ray,
                   "screen_bytes_per_launch": scr, "per_kernel_dram_bytes": avg,
                   "captured_frame_updates": frame_updates,
                   "integrate_update_bracket_bytes_per_update": bracket / frame_updates if frame_updates else None},
                  open(out, "w"), indent=1)
        return
    seen = set()
    for d in rs:
        k = d["kernel"]
        print(f"== {k}")
        for m, name in M:
            if name in d:
                v = d[name]
                print(f"   {name:24s} {v:,.1f}" if isinstance(v, float) else f"   {name:24s} {v}")
        if "global_ld_requests" in d and d.get("global_ld_requests"):
            print(f"   {'sectors_per_request':24s} {d['global_ld_sectors'] / d['global_ld_requests']:.2f}")
        if k not in seen:
            seen.add(k)
            print(f"   stalls (% of samples)    {stalls(rep, k.split('::')[-1].split('<')[0])}")


if __name__ == "__main__":
    main()
