"""Summarise ncu reports and launch lists into profiles/ (text, committed).

    python tools/summarize_ncu.py TAG [WORKLOAD] # reads gpurun_out/prof_TAG_*.ncu-rep,
                                                 # gpurun_out/launches_TAG.csv
Writes profiles/TAG_kernels.md, profiles/TAG_launches.csv (copy) and updates
profiles/traffic.json (dram bytes per launch of each profiled kernel, read by
bench.py for roofline.traffic).
"""
import csv
import glob
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
OUT = os.path.join(ROOT, "gpurun_out")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("sm__inst_executed.sum", "warp_inst"),
    ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue_active_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__cycles_active.avg", "sm_active_cyc"),
    ("gpc__cycles_elapsed.max", "elapsed_cyc"),
]

# ncu kernel -> bench.py kernel group; figures are summed over a group's kernels
KEY = {"k_blend_fused": "blend", "k_blend_bwd": "blend_bwd", "k_blend_fwd": "blend_fwd",
       "k_pre_count": "bin", "k_pre_scan": "bin", "k_pre_emit": "bin", "k_scan_tiles": "bin",
       "k_scatter_emitted": "bin", "k_tile_sort": "bin", "k_tile_sort_big": "bin",
       "k_chain_sums": "chain", "k_chain": "chain", "k_adam": "adam", "k_adam_flat": "adam"}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2:]
    res = []
    for v in vals:
        d = {}
        for name, short in METRICS:
            if name in h:
                i = h.index(name)
                try:
                    x = float(v[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if u == "Kbyte":
                    x *= 1e3
                elif u == "Mbyte":
                    x *= 1e6
                elif u == "Gbyte":
                    x *= 1e9
                elif u in ("usecond", "us"):
                    x *= 1e3
                elif u in ("nsecond", "ns"):
                    pass
                elif u in ("msecond", "ms"):
                    x *= 1e6
                d[short] = x
        d["kernel"] = v[h.index("Kernel Name")]
        res.append(d)
    return res


def main(tag, workload):
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# ncu summary, {tag}", "",
             "One `ncu --set full --clock-control none` capture per kernel of `python bench.py --steps 2 --warmup 1`",
             f"(workload `{workload}`; cold-cache, serialised replay: compare shares, not absolute times).", "",
             "| kernel | dur (us) | DRAM rd+wr (MB) | DRAM % | warp inst (M) | issue-active % (elapsed) | FMA pipe % | occupancy % | regs | SM active / elapsed |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    traffic_path = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    issue_path = os.path.join(PROF, "issue.json")
    issue = json.load(open(issue_path)) if os.path.exists(issue_path) else {}
    sums = {}
    aux = tuple(f"prof_{tag}_{wl}_" for wl in ("cfg3", "cfg4", "lidar", "window"))    # summarize_aux.py's
    for rep in sorted(glob.glob(os.path.join(OUT, f"prof_{tag}_*.ncu-rep"))):
        if os.path.basename(rep).startswith(aux):
            continue
        for d in raw(rep):
            name = d["kernel"].replace("void ", "").split("(")[0].split("::")[-1].split("<")[0]
            tb = d.get("dram_read", 0) + d.get("dram_write", 0)
            lines.append(f"| {name} | {d.get('duration', 0) / 1e3:.1f} | {tb / 1e6:.1f} | {d.get('dram_%', 0):.1f} | "
                         f"{d.get('warp_inst', 0) / 1e6:.1f} | {d.get('issue_active_%', 0):.1f} | "
                         f"{d.get('fma_pipe_%', 0):.1f} | {d.get('occupancy_%', 0):.1f} | {d.get('regs', 0):.0f} | "
                         f"{d.get('sm_active_cyc', 0) / max(d.get('elapsed_cyc', 1), 1):.2f} |")
            if name in KEY:
                grp = KEY[name]
                sums.setdefault(grp, {"traffic": 0.0, "inst": 0.0, "kernels": []})
                sums[grp]["traffic"] += tb
                sums[grp]["inst"] += d.get("warp_inst", 0)
                sums[grp]["kernels"].append(name)
    tw, iw = traffic.setdefault(workload, {}), issue.setdefault(workload, {})
    for grp, v in sums.items():
        tw[grp] = v["traffic"]
        iw[grp] = {"warp_inst_per_launch": v["inst"], "capture": tag, "kernels": sorted(v["kernels"])}
    open(os.path.join(PROF, f"{tag}_kernels.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    json.dump(issue, open(issue_path, "w"), indent=1)
    lc = os.path.join(OUT, f"launches_{tag}.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(PROF, f"{tag}_launches.csv"))
        agg = defaultdict(list)
        rows = list(csv.reader(open(lc)))
        hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
        h = rows[hi]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        for r in rows[hi + 1:]:
            v = float(r[vi].replace(",", ""))
            v = v / 1e3 if r[ui] in ("nsecond", "ns") else (v if r[ui] in ("usecond", "us") else v * 1e3)
            agg[r[ki].split("(")[0]].append(v)
        tot = sum(sum(v) for v in agg.values())
        out = ["", f"## launch list ({tag}_launches.csv): device time by kernel", "",
               "| kernel | launches | mean (us) | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            out.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")
        with open(os.path.join(PROF, f"{tag}_kernels.md"), "a") as f:
            f.write("\n".join(out) + "\n")
    print(open(os.path.join(PROF, f"{tag}_kernels.md")).read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "cfg2")
