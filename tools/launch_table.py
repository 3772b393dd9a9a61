"""Mean device time per kernel from an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_table.py gpurun_out/launches_X.csv [skip_first_n_launches]
"""
import csv
import sys
from collections import OrderedDict, defaultdict


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    h = rows[0]
    iname, imet, ival = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    t = defaultdict(list)
    order = OrderedDict()
    for r in rows[1 + skip:]:
        if r[imet] != "gpu__time_duration.sum":
            continue
        name = r[iname].split("(")[0].replace("void ", "")
        t[name].append(float(r[ival].replace(",", "")))
        order[name] = None
    tot = sum(sum(v) for v in t.values())
    for k in sorted(order, key=lambda k: -sum(t[k])):
        v = t[k]
        print(f"{k[:60]:60s} n={len(v):4d} mean={sum(v)/len(v)/1e3:9.2f} us  share={sum(v)/tot*100:5.1f}%")


if __name__ == "__main__":
    main()
