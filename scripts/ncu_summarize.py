"""Summarise ncu reports: python scripts/ncu_summarize.py out.json rep1.ncu-rep [rep2 ...]"""
import csv, io, json, subprocess, sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_peak",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_threads_per_warp_inst",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": "ld_sectors",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum": "ld_requests",
    "lts__t_requests_srcunit_tex_op_atom.sum": "l2_atom_requests",
    "smsp__inst_executed.sum": "inst_executed",
    "lts__t_requests_srcunit_tex_op_atom_dot_alu.sum": "l2_atom_alu_requests",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_active_pct",
}
UNIT = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}

# the library build the reports were captured from (scripts/prof_targets.py writes it):
# bench.py reuses counts only from summaries of its own source hash
try:
    BUILD = open("gpurun_out/build_info.txt").read().strip()
except OSError:
    BUILD = ""
out = []
for rep in sys.argv[2:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    stall_cols = [i for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        d = {"report": rep.split("/")[-1], "kernel": r[h.index("Kernel Name")][:90], "build": BUILD}
        for k, name in KEYS.items():
            if k in h:
                i = h.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[name] = v * UNIT.get(units[i], 1.0) if units[i] in UNIT else v
        stalls = []
        for i in stall_cols:
            try:
                stalls.append((float(r[i].replace(",", "")), h[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
        d["top_stalls_cycles_per_issue"] = [(n, round(v, 2)) for v, n in sorted(stalls, reverse=True)[:5]]
        if "dram_read" in d and "duration" in d:
            d["dram_bytes"] = d["dram_read"] + d.get("dram_write", 0)
            d["dram_gbs"] = d["dram_bytes"] / d["duration"] / 1e9
        out.append(d)
json.dump(out, open(sys.argv[1], "w"), indent=1)
for d in out:
    print(f'{d["kernel"][:60]:60s} {d.get("duration",0)*1e6:10.1f} us  dram {d.get("dram_bytes",0)/1e6:9.1f} MB  {d.get("dram_gbs",0):7.0f} GB/s  occ {d.get("achieved_occupancy_pct",0):5.1f}%')
