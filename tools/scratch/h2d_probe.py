"""H2D bandwidth from pinned host memory under different CPU affinities (timing aid)."""
import os, subprocess, sys, time
import torch
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
print(subprocess.run(["lscpu"], capture_output=True, text=True).stdout[-900:])
def bw(tag):
    x = torch.empty(39 * 2**20, dtype=torch.uint8).pin_memory()
    x.fill_(1)
    d = torch.empty(39 * 2**20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s): d.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    res = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s); d.copy_(x, non_blocking=True); b.record(s)
        torch.cuda.synchronize()
        res.append(39 * 2**20 / (a.elapsed_time(b) * 1e-3) / 1e9)
    res.sort()
    print(tag, "GB/s min/med/max", round(res[0], 1), round(res[10], 1), round(res[-1], 1), "cpus", len(os.sched_getaffinity(0)))
torch.cuda.init()
bw("default")
ncpu = os.cpu_count()
for part in (range(0, ncpu // 2), range(ncpu // 2, ncpu)):
    os.sched_setaffinity(0, set(part))
    bw(f"cpus {part.start}-{part.stop - 1}")
