"""Summarise tools/gpu_prof_aux.sh into profiles/ (text, committed).

    python tools/summarize_aux.py TAG

Reads gpurun_out/aux_TAG_<workload>.csv (every kernel of the bench's timed
region: device time, DRAM bytes, warp instructions) and the full captures
gpurun_out/prof_TAG_<workload>_<kernel>.ncu-rep; writes
profiles/TAG_aux_kernels.md and records, per workload, the DRAM bytes and
warp instructions per unit of the line's metric (frame / measurement /
update) in profiles/traffic.json and profiles/issue.json under the kernel
group "unit" (bench.py -> roofline.traffic of those lines).
"""
import csv
import glob
import json
import os
import shutil
import sys
from collections import OrderedDict, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
OUT = os.path.join(ROOT, "gpurun_out")
sys.path.insert(0, os.path.join(ROOT, "tools"))
from summarize_ncu import raw  # noqa: E402

# units the timed region processes (bench.py: cfg3 100 frames, window 40
# maintains, lidar --steps 3 measurements, cfg4 --steps 2 updates)
UNITS = {"cfg3": (100, "frame"), "window": (40, "maintain"), "lidar": (3, "measurement"), "cfg4": (2, "update")}
SCALE = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def read_launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, im, iu, iv, iid = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                           h.index("Metric Value"), h.index("ID"))
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        try:
            v = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        except ValueError:
            continue
        per[r[iid]][r[im]] = v
        names[r[iid]] = r[ik].split("(")[0].replace("void ", "")
    agg = OrderedDict()
    for lid, m in per.items():
        a = agg.setdefault(names[lid], defaultdict(float))
        a["n"] += 1
        a["t"] += m.get("gpu__time_duration.sum", 0.0)
        a["dram"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a["inst"] += m.get("smsp__inst_executed.sum", 0.0)
    return agg


def main(tag):
    traffic_path, issue_path = os.path.join(PROF, "traffic.json"), os.path.join(PROF, "issue.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    issue = json.load(open(issue_path)) if os.path.exists(issue_path) else {}
    lines = [f"# ncu summary, {tag}: auxiliary workloads", "",
             "Every kernel inside the bench's timed region (`ncu --nvtx --nvtx-include lsb_timed/`, metrics "
             "gpu__time_duration, dram__bytes_read/write, smsp__inst_executed; ncu serialises launches and flushes "
             "caches between them, so times are cold-cache upper bounds — compare shares).", ""]
    for wl, (units, uname) in UNITS.items():
        p = os.path.join(OUT, f"aux_{tag}_{wl}.csv")
        if not os.path.exists(p):
            continue
        shutil.copy(p, os.path.join(PROF, f"{tag}_aux_{wl}_launches.csv"))
        agg = read_launches(p)
        tt = sum(a["t"] for a in agg.values()) or 1.0
        dram = sum(a["dram"] for a in agg.values())
        inst = sum(a["inst"] for a in agg.values())
        lines += [f"## {wl} ({units} {uname}s timed)", "",
                  f"Per {uname}: {tt / units / 1e3:.1f} us of serialised kernel time, {dram / units / 1e6:.2f} MB "
                  f"DRAM, {inst / units / 1e6:.3f} M warp instructions.", "",
                  "| kernel | launches | mean (us) | share | DRAM MB / launch | warp inst (k) / launch |",
                  "|---|---|---|---|---|---|"]
        for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
            lines.append(f"| {k} | {int(a['n'])} | {a['t'] / a['n'] / 1e3:.2f} | {a['t'] / tt * 100:.1f}% | "
                         f"{a['dram'] / a['n'] / 1e6:.3f} | {a['inst'] / a['n'] / 1e3:.1f} |")
        lines.append("")
        traffic.setdefault(wl, {})["unit"] = dram / units
        issue.setdefault(wl, {})["unit"] = {"warp_inst_per_launch": inst / units, "capture": tag,
                                            "note": f"per {uname}, all kernels of the timed region"}
        for rep in sorted(glob.glob(os.path.join(OUT, f"prof_{tag}_{wl}_*.ncu-rep"))):
            for d in raw(rep):
                name = d["kernel"].replace("void ", "").split("(")[0].split("::")[-1].split("<")[0]
                tb = d.get("dram_read", 0) + d.get("dram_write", 0)
                lines.append(f"Full capture `{name}`: {d.get('duration', 0) / 1e3:.1f} us, DRAM {tb / 1e6:.2f} MB "
                             f"({d.get('dram_%', 0):.1f}% of peak), issue-active {d.get('issue_active_%', 0):.1f}%, "
                             f"occupancy {d.get('occupancy_%', 0):.1f}%, {d.get('regs', 0):.0f} regs, SM active / "
                             f"elapsed {d.get('sm_active_cyc', 0) / max(d.get('elapsed_cyc', 1), 1):.2f}.")
                lines.append("")
    open(os.path.join(PROF, f"{tag}_aux_kernels.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    json.dump(issue, open(issue_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
