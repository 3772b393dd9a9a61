"""Top warp-stall SASS instructions of an ncu capture (with their neighbours).

    python tools/sass_hot.py gpurun_out/prof_X.ncu-rep [top_n]
"""
import csv
import io
import subprocess
import sys


def main(rep, top=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = rows[2:]
    isrc, iss, ia = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    recs = [(int(r[iss] or 0), float(r[ia] or 0), k, r[isrc].strip()) for k, r in enumerate(data) if len(r) > iss]
    tot = sum(r[0] for r in recs) or 1
    print(f"{rows[0][1]}: {len(recs)} SASS, {tot} stall samples, {sum(r[1] for r in recs) / 1e6:.2f} M warp inst")
    for s, n, k, src in sorted(recs, reverse=True)[:top]:
        print(f"{s:6d} {s / tot * 100:5.1f}%  n={n / 1e3:8.1f}k  #{k:5d}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
