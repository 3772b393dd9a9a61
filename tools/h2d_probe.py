"""H2D bandwidth of this box from pinned host memory (the e2e pass copies
10 keyframe frames of 3.9 MB per step): one 3.9 MB copy, 10 back to back on
one stream, 10 round-robin on 2 / 4 streams, and one 39 MB copy.

    python tools/h2d_probe.py
"""
import json

import torch


def main():
    dev = torch.device("cuda", 0)
    nb = 1280 * 1024 * 3
    host = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(10)]
    big = torch.empty(10 * nb, dtype=torch.uint8).pin_memory()
    dst = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(10)]
    dbig = torch.empty(10 * nb, dtype=torch.uint8, device=dev)
    out = {}
    for ns in (1, 2, 4):
        streams = [torch.cuda.Stream(dev) for _ in range(ns)]
        ts = []
        for rep in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            for s in streams:
                s.wait_event(a)
            for i in range(10):
                with torch.cuda.stream(streams[i % ns]):
                    dst[i].copy_(host[i], non_blocking=True)
            for s in streams:
                torch.cuda.current_stream().wait_stream(s)
            b.record()
            torch.cuda.synchronize()
            if rep:
                ts.append(a.elapsed_time(b))
        out[f"10x3.9MB_{ns}streams_GBps"] = 10 * nb / (min(ts) * 1e-3) / 1e9
    ts = []
    for rep in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dbig.copy_(big, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        if rep:
            ts.append(a.elapsed_time(b))
    out["1x39MB_GBps"] = 10 * nb / (min(ts) * 1e-3) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
