"""Benchmark: sliding-window splat fwd+bwd+Adam on B200 (BASELINE.json config 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2] [--alpha-cut 0.00392156862745098]

One step = every keyframe view rendered (preprocess, tile binning, blend),
scored (L1 photometric loss) and back-propagated into the window's
gradient buffer, an NCCL all-reduce of that buffer when N > 1 (views sharded
v -> rank v mod N), then one Adam step in storage coordinates on all window
Gaussians.  Inputs: the reference's own synthetic room scene (sim.bake_scene
restated in paper_2501_08672_b200/scene.py), orbit keyframes, observed images
= clean renders, window = scene with SH colours perturbed U(-0.1, 0.1) (seed 0).

Prints ONE JSON line on rank 0.  `--impl reference` times the reference's CPU
algorithm (the oracle port, oracle/) on this host's cores instead.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "splat fwd+bwd Mpix/s & Gaussians/s at 1/2/4/8 B200; % HBM roofline"
CONFIGS = {
    # name: (v_s, n_views, width, height)
    # "target": the north star's 500k-Gaussian / 1280x1024 / 10-keyframe window
    # (bake_room(0.0457) = 512,808 Gaussians, the CLI orbit)
    "target": (0.0457, 10, 1280, 1024),
    "cfg1": (0.323, 1, 640, 512),
    "cfg2": (0.0723, 10, 1280, 1024),
    "cfg5": (0.0229, 64, 1920, 1080),
}
VOXEL_CFG = dict(frames=100, root_len=0.1, max_level=3, cand_stride=8)   # config 3
FALLBACK_HBM_GBS = 6650.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi's start-up takes driver locks that stall kernel
            # launches: wait for its first sample before the timed region
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.02)
        except OSError:
            self.proc = None
        # the timed region as an NVTX range: `ncu --nvtx --nvtx-include lsb_timed/`
        # profiles exactly the kernels the line's numbers come from
        import torch
        torch.cuda.nvtx.range_push("lsb_timed")
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        import torch
        torch.cuda.nvtx.range_pop()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def build_workload(cfg_name, alpha_cut):
    from tools.scene import bake_room, camera_for, orbit_views
    v_s, V, W, H = CONFIGS[cfg_name]
    means, rots, scales, opac, shs = bake_room(v_s)
    rng = np.random.default_rng(0)
    shs_win = shs.copy()
    shs_win[:, 0, :] += rng.uniform(-0.1, 0.1, size=shs_win[:, 0, :].shape)
    return dict(gt=(means, rots, scales, opac, shs), win=(means, rots, scales, opac, shs_win),
                cam=camera_for(W, H), views=orbit_views(V), V=V, W=W, H=H, N=len(means),
                alpha_cut=alpha_cut)


# ---------------------------------------------------------------- CPU legs ---
class CpuStep:
    """The reference algorithm on this host (oracle port: C + OpenMP blend,
    numpy elsewhere, all host threads), on the same window, views and frames
    as the GPU arm.  `view(v)` is one keyframe's render + L1 loss + backward,
    accumulating the mean gradient; `adam()` is the storage-coordinate Adam
    step on all window Gaussians with the accumulated gradient.  Observed
    frames are rendered from the clean scene once per view, untimed."""

    def __init__(self, wl, frames="u8"):
        from types import SimpleNamespace
        from oracle import raster as orc
        from oracle.optim import Adam, DEFAULT_CFG, adam_param_step, photometric_loss
        self.orc, self.loss, self.adam_step, self.cfg = orc, photometric_loss, adam_param_step, DEFAULT_CFG
        f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
        keys = ("means", "rots", "scales", "opacities", "shs")
        self.gt = {k: f32(v) for k, v in zip(keys, wl["gt"])}
        self.P = {k: f32(v) for k, v in zip(keys, wl["win"])}
        self.wl, self.frames, self.cam = wl, frames, wl["cam"]
        self.st = SimpleNamespace(near=0.01, dilation=0.3, alpha_clamp=0.99, transmittance_min=1e-4,
                                  footprint_sigma=6.0, alpha_cut=wl["alpha_cut"], max_footprint_px=512.0,
                                  background=np.zeros(3), sh_degree=0)
        n = len(self.P["means"])
        self.opt = Adam({"mean": (n, 3), "rot": (n, 3), "scale": (n, 3), "opacity": (n,), "sh": self.P["shs"].shape})
        self.obs = {}
        self.zero()

    def zero(self):
        n = len(self.P["means"])
        self.g = {"mean": np.zeros((n, 3)), "rot": np.zeros((n, 3)), "scale": np.zeros((n, 3)),
                  "opacity": np.zeros(n), "sh": np.zeros(self.P["shs"].shape)}

    def observed(self, v):
        if v not in self.obs:
            T_cw = self.wl["views"][v].inverse()
            o = self.orc.render(self.gt, T_cw.R, T_cw.t, self.cam, self.st)["image"]
            if self.frames == "u8":     # the same 8-bit frames the GPU arm reads, as read_ppm returns them
                o = np.clip(np.round(o * 255.0), 0, 255).astype(np.uint8).astype(np.float64) / 255.0
            self.obs[v] = o
        return self.obs[v]

    def view(self, v):
        """Seconds for view v's render + loss + backward (+ gradient accumulation)."""
        obs = self.observed(v)
        T_cw = self.wl["views"][v].inverse()
        t0 = time.perf_counter()
        c = self.orc.render(self.P, T_cw.R, T_cw.t, self.cam, self.st)
        _, _, g_img = self.loss(c["image"], obs)
        rb = self.orc.backward(c, g_img)
        for k in self.g:
            self.g[k] += rb["grads"][k] / self.wl["V"]
        return time.perf_counter() - t0

    def adam(self):
        t0 = time.perf_counter()
        self.adam_step(self.P, self.g, self.opt, self.cfg, np.zeros(len(self.P["means"]), bool))
        self.zero()
        return time.perf_counter() - t0


def workload_config(args, wl):
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": args.config, "gaussians": wl["N"], "views": wl["V"], "width": wl["W"],
            "height": wl["H"], "alpha_cut": wl["alpha_cut"],
            "frames": ("8-bit (H,W,3), u/255.0 in f64 like read_ppm" if args.frames == "u8" else "float32 (H,W,3)"),
            "l2": "GPU arm: flushed before every timed step (256 MB write outside the step's event pair)"}


def run_reference(args, wl, rank):
    """`--impl reference`: the reference's CPU algorithm (the oracle port; the
    Python reference cannot travel to the GPU box) on this host's cores.  A
    timed step is ONE keyframe view (view i mod V: render + L1 loss +
    backward), and every V-th step also runs the Adam step over all window
    Gaussians with the accumulated mean gradient - so V consecutive steps are
    one full window step and `value` = pixels processed / time spent."""
    if rank != 0:
        return
    V, P_px = wl["V"], wl["W"] * wl["H"]
    cs = CpuStep(wl, args.frames)
    for v in range(V):
        cs.observed(v)                  # observed frames: untimed set-up
    times = []
    for i in range(args.warmup + args.steps):
        v = i % V
        t = cs.view(v)
        if v == V - 1:
            t += cs.adam()
        if i >= args.warmup:
            times.append(t)
    t = float(np.mean(times))
    value = P_px / t / 1e6
    sample = (f"each step = one keyframe view (render + L1 loss + backward, {wl['W']}x{wl['H']}, {wl['N']} "
              f"Gaussians, alpha_cut={wl['alpha_cut']:.6g}), views in turn, + the Adam step over all window "
              f"Gaussians on every {V}-th step ({sum(1 for i in range(args.warmup, args.warmup + args.steps) if i % V == V - 1)}"
              f" Adam steps timed); oracle port, {os.cpu_count()} host threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Mpix/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "step_unit": f"one keyframe view (+ Adam every {V}-th step); {V} steps = one window step",
        "gaussians_per_s": wl["N"] / t,
        "parallelism": f"cpu threads ({os.cpu_count()})",
        "config": workload_config(args, wl),
        "cpu_baseline": {"value": value, "unit": "Mpix/s", "cores": os.cpu_count(), "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "Mpix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- GPU leg ----
def algorithmic_bytes(N, K, M, I, P, pbytes=8, obytes=4):
    """Per-launch algorithmic HBM bytes.  pbytes: bytes per
    parameter of the working copy (8: the f64 copy optimize_window steps);
    obytes: bytes per observed channel (1 for 8-bit frames, 4 for f32)."""
    ob = 3 * obytes
    prm = pbytes * (16 + 3 * K)     # one Gaussian's parameters
    grd = 4 * (10 + 3 * K)          # one Gaussian's gradient row (f32)
    mom = pbytes * (10 + 3 * K)     # one Gaussian's Adam moment row
    return {
        "bin": N * prm + M * (64 + 8 + 4) + I * (4 + 4 + 4 + 8 + 4 + 4),
        "blend_fwd": I * (64 + 4) + P * (12 + 4 + 4 + ob + 12),   # + fused loss: read observed, write dL/dI
        "blend_bwd": I * (64 + 4 + 4 + 36) + P * (12 + 12 + 4),
        # fused forward + loss + backward: records and slots read by both walks,
        # intersection ids, partials written; observed read (no image round trip)
        "blend": I * (64 + 4 + 64 + 4 + 4 + 36) + P * ob,
        "chain": M * (64 + 4 + prm + 2 * grd) + I * 36,
        "adam": N * (2 * prm + grd + 4 * mom + 1),
    }


def profile_figure(name, workload, kernel):
    """profiles/<name> is {workload: {kernel: figure}} (one ncu capture per workload)."""
    p = os.path.join(ROOT, "profiles", name)
    if not os.path.exists(p):
        return None
    return json.load(open(p)).get(workload, {}).get(kernel)


AUX_TRAFFIC_NOTE = ("ncu dram__bytes_read + write summed over every kernel of the timed region (NVTX lsb_timed; "
                    "cold caches between launches; profiles/r02c_aux_kernels.md)")


def survey_step_bytes(N, K, counts, bands, W):
    """SURVEY.md §8(d) as written: B_step = 504 N + sum_v (420 M_v + 12 I_v + 52 P_v)
    (its K = 1 figures: 64 B of parameters, 52 B of gradient / moment rows)."""
    assert K == 1, "the survey's step model is stated for SH degree 0"
    return 504 * N + sum(420 * c[0] + 12 * c[1] + 52 * W * (y1 - y0) for c, (y0, y1) in zip(counts, bands))


def run_ours(args, wl, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2501_08672_b200.optimize import OptimConfig, WindowEngine
    from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    settings = RasterSettings(alpha_cut=wl["alpha_cut"])
    V, W, H, N = wl["V"], wl["W"], wl["H"], wl["N"]
    gt = GaussianArrays(*wl["gt"], device=dev)
    win = GaussianArrays(*wl["win"], device=dev)
    # this rank's render units: whole views (v -> rank v mod N), or row bands
    # of the views when N does not divide them (dist.shard_units: config 2's
    # 10 views become 20 half views at N = 4, 40 quarter views at N = 8)
    from paper_2501_08672_b200.dist import shard_units_mixed as shard_units
    units = shard_units(V, world, rank, H)
    my_views = [u[0] for u in units]
    bands = [(u[1], u[2]) for u in units]
    frames = {v: render(gt, wl["views"][v], wl["cam"], settings, retain_cache=False).image.clone()
              for v in sorted(set(my_views))}
    if args.frames == "u8":
        # the camera's 8-bit frames, quantised the way write_ppm stores them
        # (raster.py:511-517); the kernels read u / 255.0 like read_ppm
        frames = {v: torch.clamp(torch.round(o.double() * 255.0), 0, 255).to(torch.uint8) for v, o in frames.items()}
    observed = [frames[v][y0:y1].contiguous() for v, y0, y1 in units]
    del gt, frames
    # L2 flush between timed steps: a write larger than the 126 MB L2, issued
    # outside each step's event pair
    flush_buf = torch.empty(64 * 2 ** 20, dtype=torch.int32, device=dev)
    spreads = []

    def timed(run_one):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        with torch.cuda.stream(stream):
            for a, b in evs:
                flush_buf.zero_()
                a.record(stream)
                run_one()
                b.record(stream)
        torch.cuda.synchronize()
        # the median step; the spread is kept for the JSON line
        ts = [a.elapsed_time(b) for a, b in evs]
        spreads.append((float(np.min(ts)), float(np.max(ts))))
        return float(np.median(ts))
    stream = torch.cuda.Stream(dev)
    eng = WindowEngine(win, wl["cam"], [wl["views"][v] for v in my_views], settings, OptimConfig(),
                       n_views_total=V, stream=stream, lanes=args.lanes, bands=bands)
    counts = []
    for v in range(len(my_views)):      # per-unit M, I for the byte model
        T = eng.views[v]
        eng.state.set_pose(T.R, T.t)
        eng.state.set_camera(eng.view_cams[v])
        from paper_2501_08672_b200.raster import render_bin
        render_bin(eng.state, stream)
        counts.append(eng.state.read_counts(stream)[:2])
    # the engine's exchange: bucketed async all-reduce (mean | rot | scale +
    # opacity | sh), Adam stepping each bucket as soon as it is reduced
    from paper_2501_08672_b200.dist import make_allreduce
    allreduce = make_allreduce() if world > 1 else None
    exchange = "nccl"
    if world > 1 and args.exchange == "p2p":
        # fused gradient exchange + Adam over NVLink peer memory (dist.PeerExchange);
        # every rank falls back to NCCL if any rank cannot set it up
        ok = 1
        try:
            from paper_2501_08672_b200.dist import PeerExchange
            eng.exchange = PeerExchange(eng)
        except Exception as exc:          # noqa: BLE001
            ok = 0
            print(f"[bench] rank {rank}: peer exchange unavailable ({exc}); NCCL all-reduce", file=sys.stderr)
        t = torch.tensor([ok], device=dev, dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if int(t.item()):
            exchange = "p2p"
        else:
            eng.exchange = None

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            eng.step(observed, allreduce=allreduce)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    smi_index = int(vis.split(",")[local_rank]) if vis and vis.split(",")[local_rank].isdigit() else local_rank

    # pass 1 (kernel timing): a one-lane engine on the same window, eager
    # launches serialised on one stream with CUDA events around every kernel,
    # so each kernel's duration is its own (not shared with a concurrent lane)
    timers: dict = {}
    keng = WindowEngine(win, wl["cam"], [wl["views"][v] for v in my_views], settings, OptimConfig(),
                        n_views_total=V, stream=stream, lanes=1, isect_cap=eng.lanes[0].state.dims.isect_cap,
                        bands=bands)
    with torch.cuda.stream(stream):
        keng.step(observed, allreduce=allreduce)
    eager_ms = timed(lambda: keng.step(observed, allreduce=allreduce, timers=timers))
    del keng

    # pass 2 (the headline): the same step captured once as a CUDA graph (the
    # NCCL all-reduce included when N > 1; if any rank fails to capture, all
    # ranks fall back to eager launches)
    def try_capture(obs):
        ok = 1
        try:
            eng.capture(obs, allreduce)
            with torch.cuda.stream(stream):
                eng.replay()
            torch.cuda.synchronize()
        except Exception as exc:          # noqa: BLE001 - fall back to eager
            ok = 0
            eng.graph = None
            print(f"[bench] rank {rank}: CUDA-graph capture failed ({exc}); eager launches", file=sys.stderr)
        if world > 1:
            t = torch.tensor([ok], device=dev, dtype=torch.int32)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            ok = int(t.item())
            if not ok:
                eng.graph = None
        return bool(ok)

    use_graph = bool(args.graph) and try_capture(observed)
    graph_headline = use_graph
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(smi_index) as clk:
        ms = timed(lambda: eng.replay() if use_graph else eng.step(observed, allreduce=allreduce))
    with torch.cuda.stream(stream):
        eng.finish()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    assert eng.check_capacity(), "intersection capacity exceeded during the timed region"
    losses = eng.losses()

    # per-kernel device time inside the timed region (event pairs on `stream`)
    ktime = {k: [ev[i].elapsed_time(ev[i + 1]) for i in range(0, len(ev), 2)] for k, ev in timers.items()}
    M_avg = float(np.mean([c[0] for c in counts])) if counts else 0.0
    I_avg = float(np.mean([c[1] for c in counts])) if counts else 0.0
    K = int(win.shs.shape[1])
    P_avg = float(np.mean([W * (y1 - y0) for y0, y1 in bands]))
    ab = algorithmic_bytes(N, K, M_avg, I_avg, P_avg, pbytes=eng.arrays.means.element_size(),
                           obytes=observed[0].element_size())
    per_step_ms = {k: float(np.sum(v)) / args.steps for k, v in ktime.items()}
    dom = max(("bin", "blend", "blend_fwd", "blend_bwd", "chain"), key=lambda k: per_step_ms.get(k, 0.0))
    dom_ms = float(np.mean(ktime[dom]))
    hbm, hbm_src = peaks()
    achieved = ab[dom] / (dom_ms * 1e-3) / 1e9
    # ncu figures of the same kernel on the same workload (profiles/*.json are
    # keyed by workload; another workload's capture is never attached)
    traffic = profile_figure("traffic.json", args.config, dom)
    issue = profile_figure("issue.json", args.config, dom)
    # bytes of the kernels that ran in the timed step, each at its launch count
    nlaunch = {k: len(v) // args.steps for k, v in ktime.items()}
    ran_bytes = sum(ab[k] * nlaunch[k] for k in nlaunch)
    # SURVEY.md §8(d)'s step model: B_step = 504 N + sum_v (420 M_v + 12 I_v + 52 P)
    survey_bytes = survey_step_bytes(N, K, counts, bands, W)

    # end-to-end through the public API with host buffers: every step copies
    # this rank's observed images from pinned host memory (copy stream, in
    # view order, overlapping the lanes' kernels) and reads the loss sums back
    host_obs = [o.cpu().pin_memory() for o in observed]
    eng.copy_streams = max(1, args.copy_streams)
    with torch.cuda.stream(stream):
        eng.step(host_obs, allreduce=allreduce)            # e2e warm-up (staging buffers)
    torch.cuda.synchronize()
    if use_graph:
        use_graph = try_capture(host_obs)
    def e2e_step():
        if use_graph:
            eng.replay()
        else:
            eng.step(host_obs, allreduce=allreduce)
        _ = eng.loss.sums().to("cpu", non_blocking=False)

    e_ms = timed(e2e_step)
    if world > 1:
        t = torch.tensor([e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    h2d = sum(o.numel() * o.element_size() for o in observed)
    d2h = int(eng.loss.sums().numel() * 8)
    # this box's host -> device bandwidth for the same pinned frames (untimed;
    # the e2e step is copy-bound when it cannot move h2d bytes within a step)
    dst = [torch.empty_like(o, device=dev) for o in observed]
    bw = []
    for _ in range(3):
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record()
        for d_, h_ in zip(dst, host_obs):
            d_.copy_(h_, non_blocking=True)
        b_ev.record()
        torch.cuda.synchronize()
        bw.append(h2d / (a_ev.elapsed_time(b_ev) * 1e-3) / 1e9)
    h2d_gbps = float(max(bw))
    del dst

    clk_sum = clk.summary()
    if rank == 0:
        value = V * W * H / (ms * 1e-3) / 1e6
        out = {
            "metric": METRIC, "value": value, "unit": "Mpix/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "gaussians_per_s": V * N / (ms * 1e-3),
            "visible_splats_per_s": float(sum(c[0] for c in counts)) * world / (ms * 1e-3),
            "parallelism": f"view-sharded dp{world}",
            "config": workload_config(args, wl),
            "details": {"view_lanes": args.lanes, "exchange": exchange if world > 1 else None,
                       # render units per rank (dist.shard_units_mixed): whole views first,
                       # row bands of the leftover views when N does not divide the views
                       "units_per_rank": [shard_units(V, world, r, H) for r in range(world)],
                       "pixel_row_imbalance": max(sum(y1 - y0 for _, y0, y1 in shard_units(V, world, r, H))
                                                  for r in range(world)) / (V * H / world),
                       "cuda_graph": graph_headline, "cuda_graph_e2e": use_graph,
                       "serial_ms_per_step": eager_ms,
                       "kernel_timing": "separate one-lane eager pass of the same steps, events around each kernel",
                       "timing": "CUDA events around each step on the launching stream, median over steps",
                       "step_ms_min_max": {"serial": spreads[0], "headline": spreads[1],
                                           "e2e": spreads[2] if len(spreads) > 2 else None},
                       "loss_last_step": float(np.mean(losses))},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "peak_source": hbm_src,
                         "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                         "algorithmic_bytes_per_launch": ab[dom], "avg_launch_ms": dom_ms,
                         "note": "the blend is compute-side bound (SURVEY.md §8(d)): its records, lists and frame stay in L2; see issue_roofline and profiles/README.md (dependency latency at 3.7 warps per scheduler)"},
            "issue_roofline": None if not issue else {
                "kernel": dom, "unit": "warp-inst/s", "warp_inst_per_launch": issue["warp_inst_per_launch"],
                "achieved": issue["warp_inst_per_launch"] / (dom_ms * 1e-3),
                "peak": 148 * 4 * (clk_sum["sm_mhz"] or 1965.0) * 1e6,
                "frac": issue["warp_inst_per_launch"] / (dom_ms * 1e-3) / (148 * 4 * (clk_sum["sm_mhz"] or 1965.0) * 1e6),
                "source": f"ncu capture {issue.get('capture')} (one {args.config} view), live launch time"},
            "step_roofline": {
                "survey_bytes_per_step_rank0": survey_bytes,
                "survey_frac": survey_bytes / (ms * 1e-3) / 1e9 / hbm,
                "survey_model": "SURVEY.md §8(d): 504 N + sum_v (420 M_v + 12 I_v + 52 P) (f32, K=1 form)",
                "kernel_bytes_per_step_rank0": ran_bytes,
                "kernel_frac": ran_bytes / (ms * 1e-3) / 1e9 / hbm,
                "kernel_model": "algorithmic_bytes() of the kernels that ran, x their launches per step",
                "launches_per_step": nlaunch},
            "kernel_ms_per_step": per_step_ms,
            "counts_per_unit": {"visible_M": M_avg, "intersections_I": I_avg, "pixels": P_avg},
            "clocks": clk_sum,
            "e2e": {"value": V * W * H / (e_ms * 1e-3) / 1e6, "unit": "Mpix/s",
                    "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world, "ms_per_step": e_ms,
                    "h2d_GBps_measured": h2d_gbps,
                    "note": "frames copied on one copy stream in view order, each view's blend waits for its own "
                            "copy; at h2d_GBps_measured the copies take h2d_bytes / bandwidth per step"},
            "gpu_launches": args.steps * (len(my_views) * (12 if wl["alpha_cut"] > 0 and N >= 65536 else 11) + 2),
            # per view: preprocess count / scan / emit, tile scan, band search (alpha_cut > 0, N >= 65536: preprocess.cu
            # LSB_BAND_SPLAT_MIN_N), scatter, tile
            # sort, big-tile sort, fused blend (fwd + loss + bwd), loss total, chain partial sums, chain;
            # + adam and step counter per step (profiles/r02p_launches.csv)
        }
        if world == 1 and not args.no_cpu_baseline:
            cs = CpuStep(wl, args.frames)
            nv = min(2, V)
            tv = [cs.view(v) for v in range(nv)]
            ta = cs.adam()
            t_cpu = sum(tv) + ta
            out["cpu_baseline"] = {
                "value": nv * W * H / t_cpu / 1e6, "unit": "Mpix/s", "cores": os.cpu_count(), "kind": "port",
                "sample": f"views 0..{nv - 1} of {V} (render + L1 + backward) + one Adam step over all {N} window "
                          f"Gaussians on the oracle port ({t_cpu:.2f} s); value = {nv} views' pixels / that time"}
        print(json.dumps(out), flush=True)


# ------------------------------------------------------------- config 3 -----
def run_voxel(args, rank, world, local_rank):
    """Hash-octree voxel map: per frame, accumulate a 100k-point LiDAR scan
    into the leaf statistics (creating leaves), try-insert one candidate
    Gaussian per 8 points (capacity-1 leaves) and enumerate the FoV leaves
    under the scan's root voxels (pipeline.py:180-191).  Replicas only: one
    scan per frame has a single writer."""
    import ctypes
    import torch
    from paper_2501_08672_b200 import _lib
    from tools.scene import T_LI, lidar_scan, orbit_imu_pose, room_triangles, scan_directions
    from paper_2501_08672_b200.voxmap import HashOctree
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    F = VOXEL_CFG["frames"]
    tris, dirs = room_triangles(), scan_directions()
    poses = [orbit_imu_pose(a) @ T_LI for a in np.linspace(0.0, 1.5 * np.pi, F)]
    scans = [lidar_scan(T, tris, dirs, device=dev).contiguous() for T in poses]
    n_pts = [s.shape[0] for s in scans]
    cands = [s[:: VOXEL_CFG["cand_stride"]].contiguous() for s in scans]
    lib = _lib.load()
    stream = torch.cuda.current_stream()

    rcap = 1 << 18
    rset = torch.empty(rcap, dtype=torch.int64, device=dev)
    n_out = torch.zeros(1, dtype=torch.int64, device=dev)
    slots = torch.empty(max(n_pts), dtype=torch.int64, device=dev)
    cslots = torch.empty(max(c.shape[0] for c in cands), dtype=torch.int64, device=dev)
    status = torch.empty_like(cslots, dtype=torch.int32)
    out = torch.empty((1 << 23, 3), dtype=torch.int64, device=dev)

    nb = ctypes.c_size_t()
    lib.lsb_voxmap_accumulate_temp_bytes(max(n_pts), ctypes.byref(nb))
    acc_tmp = torch.empty(nb.value, dtype=torch.uint8, device=dev)

    def run(m, frames):
        st = m.struct()
        gid = 0
        for f in frames:
            p, c = scans[f], cands[f]
            # deterministic leaf statistics: stable device radix sort by leaf, one add per leaf
            lib.lsb_voxmap_accumulate(ctypes.byref(st), ctypes.c_void_p(p.data_ptr()), p.shape[0],
                                      ctypes.c_void_p(slots.data_ptr()), ctypes.c_void_p(acc_tmp.data_ptr()),
                                      acc_tmp.numel(), _lib.stream_ptr())
            lib.lsb_voxmap_try_insert(ctypes.byref(st), ctypes.c_void_p(c.data_ptr()), c.shape[0], gid,
                                      ctypes.c_void_p(cslots.data_ptr()), ctypes.c_void_p(status.data_ptr()),
                                      _lib.stream_ptr())
            gid += c.shape[0]
            lib.lsb_voxmap_fov(ctypes.byref(st), ctypes.c_void_p(p.data_ptr()), p.shape[0],
                               ctypes.c_void_p(rset.data_ptr()), rcap, ctypes.c_void_p(out.data_ptr()),
                               ctypes.c_void_p(n_out.data_ptr()), m.cap, _lib.stream_ptr())
        return n_out

    warm = HashOctree(VOXEL_CFG["root_len"], VOXEL_CFG["max_level"], capacity=1 << 23, device=dev)
    run(warm, range(min(args.warmup, F)))
    torch.cuda.synchronize()
    m = HashOctree(VOXEL_CFG["root_len"], VOXEL_CFG["max_level"], capacity=1 << 23, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        n_out = run(m, range(F))
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    assert int(m.flags.item()) == 0, "voxel table overflow"
    leaves, fov = int(m.n_used.item()), int(n_out.item())
    total_pts = sum(n_pts)
    # byte model: 12 n_pts + 168 g + 8 n_fov per frame, g the
    # leaves a frame's scan touches (key 8 + statistics read-modify-write 2 x 80)
    # and n_fov the FoV leaves it lists - counted in an untimed replay
    from paper_2501_08672_b200.sort import segments, sort_pairs
    from paper_2501_08672_b200.voxmap import keys_of_points_dev
    from paper_2501_08672_b200.window import order_keys
    rep = HashOctree(VOXEL_CFG["root_len"], VOXEL_CFG["max_level"], capacity=1 << 23, device=dev)
    g_tot, fov_tot = 0, 0
    for f in range(F):
        g_tot += int(segments(sort_pairs(order_keys(keys_of_points_dev(scans[f], rep.leaf_len, dev)), key_bits=63,
                                         signed=False)[0]).numel())
        fov_tot += int(run(rep, [f]).item())
    vox_bytes = 12 * total_pts + 168 * g_tot + 8 * fov_tot
    hbm, hbm_src = peaks()
    vox_gbs = vox_bytes / (ms * 1e-3) / 1e9
    # CPU baseline: the oracle's dict map on the first frames of the same scans
    from oracle.voxmap import Map
    om = Map(VOXEL_CFG["root_len"], VOXEL_CFG["max_level"])
    nb = 2
    t0 = time.perf_counter()
    for f in range(nb):
        p = scans[f].cpu().numpy()
        om.accumulate_points(p)
        for q in cands[f].cpu().numpy():
            om.try_insert(q)
        om.leaf_keys_under_roots({tuple(k) for k in np.floor(p / VOXEL_CFG["root_len"]).astype(np.int64)})
    t_cpu = (time.perf_counter() - t0) / nb
    if rank == 0:
        print(json.dumps({
            "metric": "voxel map insert+lookup Mpts/s (config 3)", "value": total_pts / (ms * 1e-3) / 1e6,
            "unit": "Mpts/s", "n_gpus": 1, "steps": F, "warmup": args.warmup, "ms_per_step": ms / F,
            "higher_is_better": True, "scaling": "replicas", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "cfg3", "frames": F, "points_per_frame": int(np.mean(n_pts)),
                                            "root_len": VOXEL_CFG["root_len"], "max_level": VOXEL_CFG["max_level"],
                                            "leaves_after": leaves, "fov_leaves_last": fov},
            "clocks": clk.summary(),
            # per frame: insert, slot keys, 3 radix passes x 3, segments x 3, run sums; claim / commit x 2;
            # FoV roots + leaves
            "gpu_launches": F * 20,
            "roofline": {"bound": "hbm", "kernel": "whole frame (accumulate + try_insert + FoV)",
                         "achieved": vox_gbs, "peak": hbm, "peak_source": hbm_src, "unit": "GB/s",
                         "frac": vox_gbs / hbm, "traffic": profile_figure("traffic.json", "cfg3", "unit"),
                         "traffic_note": AUX_TRAFFIC_NOTE + " per frame",
                         "algorithmic_bytes_per_frame": vox_bytes / F,
                         "model": "SURVEY.md §8(d): 12 n_pts + 168 g + 8 n_fov per frame",
                         "g_per_frame": g_tot / F, "n_fov_per_frame": fov_tot / F},
            "cpu_baseline": {"value": int(np.mean(n_pts[:nb])) / t_cpu / 1e6, "unit": "Mpts/s", "cores": 1,
                             "kind": "port", "sample": f"{nb} frames on the oracle's dict map"},
        }), flush=True)


# ------------------------------------------------------------- window -------
WINDOW_CFG = dict(frames=40, root_len=0.1, max_level=2, capacity=200_000)


def run_window(args, rank, world, local_rank):
    """Sliding-window maintenance (window.py:236-276):
    per frame, the FoV leaves of an orbit LiDAR scan are diffed against the
    live window, departing rows are written back to the map store, the
    window is compacted and the arriving leaves' Gaussians appended (capacity
    drops ranked by distance to the sensor).  The map (one Gaussian per leaf
    of all scans) and each frame's FoV key set are built before the timed
    region; the timed region is the maintain calls (host wall clock around
    each, synchronised: maintain reads its counts back).  Replicas only."""
    import torch
    from tools.scene import T_LI, lidar_scan, orbit_imu_pose, room_triangles, scan_directions
    from paper_2501_08672_b200.voxmap import HashOctree
    from paper_2501_08672_b200.window import GaussianWindow
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    F, K = WINDOW_CFG["frames"], 1
    tris, dirs = room_triangles(), scan_directions()
    poses = [orbit_imu_pose(a) @ T_LI for a in np.linspace(0.0, 1.5 * np.pi, F)]
    scans = [lidar_scan(T, tris, dirs, device=dev).contiguous() for T in poses]
    vmap = HashOctree(WINDOW_CFG["root_len"], WINDOW_CFG["max_level"], capacity=1 << 22, device=dev)
    for p in scans:
        vmap.accumulate_points_dev(p)
    keys, _ = vmap.dump_dev()
    leaf = vmap.leaf_len
    rows = torch.zeros((keys.shape[0], 16 + 3 * K), dtype=torch.float32, device=dev)
    rows[:, 0:3] = ((keys.to(torch.float64) + 0.5) * leaf).to(torch.float32)
    rows[:, 3] = rows[:, 7] = rows[:, 11] = 1.0
    rows[:, 12:15] = leaf / 2
    rows[:, 15] = 0.5
    rows[:, 16:] = torch.rand((keys.shape[0], 3 * K), generator=torch.Generator(device=dev).manual_seed(0),
                              device=dev) - 0.5
    vmap.set_gaussians_dev(keys, rows)
    fovs = [vmap.fov_leaf_keys_dev(p).clone() for p in scans]
    sensors = [np.asarray(T.t, dtype=np.float64) for T in poses]

    def walk(win, frames):
        times, reps = [], []
        for f in frames:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reps.append(win.maintain(vmap, fovs[f], sensor_pos=sensors[f]))
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        return times, reps

    walk(GaussianWindow(WINDOW_CFG["capacity"], K, device=dev), range(min(args.warmup, F)))
    with ClockSampler(local_rank) as clk:
        times, reps = walk(GaussianWindow(WINDOW_CFG["capacity"], K, device=dev), range(F))
    ms = float(np.median(times)) * 1e3
    fov_avg = float(np.mean([f.shape[0] for f in fovs]))
    win_bytes = 16 * fov_avg + 152 * float(np.mean([r.removed + r.moved + r.added for r in reps[1:]]))
    # CPU baseline: the oracle restatement (dict map) on the first frames
    from oracle.window import Window
    store = {tuple(int(v) for v in k): r for k, r in zip(keys.cpu().numpy(), rows.cpu().numpy())}
    ow = Window(WINDOW_CFG["capacity"], 16 + 3 * K)
    nb = 3
    t_cpu = []
    for f in range(nb):
        fov = {tuple(int(v) for v in k) for k in fovs[f].cpu().numpy()}
        t0 = time.perf_counter()
        ow.maintain(store, fov, leaf, None, sensors[f])
        t_cpu.append(time.perf_counter() - t0)
    if rank == 0:
        print(json.dumps({
            "metric": "sliding-window maintain ms/frame (SURVEY.md §8(f) rank 1)", "value": ms, "unit": "ms/frame",
            "n_gpus": 1, "steps": F, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "replicas", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "window", "frames": F, "root_len": WINDOW_CFG["root_len"],
                       "max_level": WINDOW_CFG["max_level"], "capacity": WINDOW_CFG["capacity"],
                       "map_gaussians": int(keys.shape[0]), "fov_keys_avg": fov_avg,
                       "added_avg": float(np.mean([r.added for r in reps[1:]])),
                       "removed_avg": float(np.mean([r.removed for r in reps[1:]])),
                       "moved_avg": float(np.mean([r.moved for r in reps[1:]])),
                       "dropped_avg": float(np.mean([r.dropped for r in reps[1:]])),
                       "timing": "host wall clock per maintain (synchronised), median over frames"},
            "clocks": clk.summary(),
            "roofline": {"bound": "hbm", "kernel": "maintain (diff, write-back, compaction, append)", "unit": "GB/s",
                         "achieved": win_bytes / (ms * 1e-3) / 1e9, "peak": peaks()[0], "peak_source": peaks()[1],
                         "frac": win_bytes / (ms * 1e-3) / 1e9 / peaks()[0],
                         "traffic": profile_figure("traffic.json", "window", "unit"),
                         "traffic_note": AUX_TRAFFIC_NOTE + " per maintain",
                         "algorithmic_bytes_per_frame": win_bytes,
                         "model": "16 n_fov (FoV keys in, diff marks) + 152 (removed + moved + added) (f32 row "
                                  "read + write)",
                         "note": "a few host syncs per frame (counts): latency bound"},
            "cpu_baseline": {"value": float(np.median(t_cpu)) * 1e3, "unit": "ms/frame", "cores": 1, "kind": "port",
                             "sample": f"first {nb} frames on the oracle restatement (dict map)"},
        }), flush=True)


# ------------------------------------------------------------- lidar --------
def run_lidar(args, rank, world, local_rank):
    """LiDAR point-to-plane measurement (SURVEY.md §8(f) rank 2,
    estimator.py:190-238): a 100k-point scan is transformed, keyed, fitted
    against its leaf's 7-neighbour plane and gated on the device, then the
    pose block of H^T R^-1 H and H^T R^-1 z is reduced on the device
    (Measurement.hb).  The map (root 0.1 m, max_level 3) holds 20 earlier
    orbit scans.  Host wall clock per measurement + reduction, synchronised.
    Replicas only (one scan per update)."""
    import torch
    from paper_2501_08672_b200.estimator import FilterConfig, NavState, lidar_measurement
    from paper_2501_08672_b200.geometry import SE3
    from tools.scene import T_LI, lidar_scan, orbit_imu_pose, room_triangles, scan_directions
    from paper_2501_08672_b200.voxmap import HashOctree
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    tris, dirs = room_triangles(), scan_directions()
    vmap = HashOctree(0.1, 3, capacity=1 << 22, device=dev)
    for a in np.linspace(0.0, 1.5 * np.pi, 20):
        vmap.accumulate_points_dev(lidar_scan(orbit_imu_pose(a) @ T_LI, tris, dirs, device=dev))
    T_wi = orbit_imu_pose(0.77)
    scan_w = lidar_scan(T_wi @ T_LI, tris, dirs, device=dev)
    T_wl = T_wi @ T_LI
    pts_l = ((scan_w - torch.as_tensor(T_wl.t, device=dev)) @ torch.as_tensor(T_wl.R, device=dev)).contiguous()
    state = NavState(SE3(T_wi.R, T_wi.t + np.array([0.01, -0.005, 0.004])))
    cfg = FilterConfig()
    for _ in range(args.warmup):
        lidar_measurement(state, pts_l, vmap, T_LI, cfg).hb()
    times = []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            meas = lidar_measurement(state, pts_l, vmap, T_LI, cfg)
            meas.hb()
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
    ms = float(np.median(times)) * 1e3
    n = int(pts_l.shape[0])
    # CPU baseline: the restatement (numpy) on the same scan and map points
    from oracle import lidar as orl
    allpts = torch.cat([lidar_scan(orbit_imu_pose(a) @ T_LI, tris, dirs, device=dev)
                        for a in np.linspace(0.0, 1.5 * np.pi, 20)]).cpu().numpy()
    stats = orl.leaf_stats(allpts, vmap.leaf_len)
    t0 = time.perf_counter()
    z, H, _ = orl.lidar_measurement(stats, vmap.leaf_len, pts_l.cpu().numpy(), T_LI.R, T_LI.t, state.T_WI.R,
                                    state.T_WI.t, cfg.lidar_gate)
    _ = H.T @ H, H.T @ z
    t_cpu = time.perf_counter() - t0
    if rank == 0:
        print(json.dumps({
            "metric": "LiDAR point-to-plane rows + H/b, Mpts/s (SURVEY.md §8(f) rank 2)", "value": n / (ms * 1e-3) / 1e6,
            "unit": "Mpts/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "replicas", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "roofline": {"bound": "hbm", "kernel": "measurement + H/b", "unit": "GB/s",
                         "achieved": 640 * n / (ms * 1e-3) / 1e9, "peak": peaks()[0], "peak_source": peaks()[1],
                         "frac": 640 * n / (ms * 1e-3) / 1e9 / peaks()[0],
                         "traffic": profile_figure("traffic.json", "lidar", "unit"),
                         "traffic_note": AUX_TRAFFIC_NOTE + " per measurement",
                         "model": "640 B per scan point: point 24 + 7 leaf statistics x 80 + z / row 56",
                         "note": "host-synchronised measurement (one read-back): latency bound"},
            "config": {"workload": "lidar", "scan_points": n, "rows_kept": int(len(meas.z)), "root_len": 0.1,
                       "max_level": 3, "map_scans": 20,
                       "timing": "host wall clock per measurement + device H/b (synchronised), median"},
            "clocks": clk.summary(),
            "cpu_baseline": {"value": n / t_cpu / 1e6, "unit": "Mpts/s", "cores": 1, "kind": "port",
                             "sample": "one full measurement on the numpy restatement (plane fits per unique leaf)"},
        }), flush=True)


# ------------------------------------------------------------- config 4 -----
def run_ieskf(args, rank, world, local_rank):
    """IESKF photometric update (config 4): 5 iterations, each re-rendering
    the 500k-Gaussian window at the running estimate, selecting semi-dense
    pixels, gating residuals, computing the pose rows and reducing
    H^T R^-1 H / H^T R^-1 z on the device; the 15x15 update on the host.
    Replicas only (one view per update)."""
    import torch
    from paper_2501_08672_b200.estimator import FilterConfig, NavState, ieskf_visual_update
    from paper_2501_08672_b200.geometry import SE3, so3_exp
    from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render
    from tools.scene import T_IC, bake_room, camera_for, orbit_imu_pose
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    means, rots, scales, opac, shs = bake_room(0.0457)
    arrays = GaussianArrays(means, rots, scales, opac, shs, device=dev)
    cam = camera_for(1280, 1024)
    st = RasterSettings(alpha_cut=args.alpha_cut)
    T_wi = orbit_imu_pose(0.5 * np.pi)
    observed = render(arrays, T_wi @ T_IC, cam, st, retain_cache=False).image.clone()
    prior = NavState(SE3(T_wi.R @ so3_exp([0.002, -0.001, 0.003]), T_wi.t + np.array([0.01, -0.005, 0.004])))
    cov0 = np.diag(np.concatenate([np.full(3, 1e-8), np.full(3, 1e-8), np.full(3, 1e-6), np.full(3, 1e-8),
                                   np.full(3, 1e-6)]))
    fcfg = FilterConfig()
    iters = 5
    for _ in range(args.warmup):
        ieskf_visual_update(prior, cov0, observed, arrays, cam, T_IC, fcfg, st, max_iter=iters, step_tol=0.0)
    torch.cuda.synchronize()
    times = []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            t0 = time.perf_counter()
            post, _ = ieskf_visual_update(prior, cov0, observed, arrays, cam, T_IC, fcfg, st, max_iter=iters,
                                          step_tol=0.0)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
    ms = float(np.median(times)) * 1e3
    err_t = float(np.abs(post.T_WI.t - T_wi.t).max())
    # per-iteration bytes: the render at the estimate (preprocess + binning + the
    # counted forward, f32 parameters and f32 observed frame), the semi-dense
    # selection (observed + T) and the pose rows / H-b (selected pixels' tile
    # lists are a small fraction); counts from one render at the prior
    from paper_2501_08672_b200.raster import render as _render
    T_wc0 = prior.T_WI @ T_IC
    out0 = _render(arrays, T_wc0, cam, st, bin_mode=1)
    M0, I0 = out0.cache.counts[0], out0.cache.counts[1]
    ab = algorithmic_bytes(len(means), int(shs.shape[1]), M0, I0, 1280 * 1024, pbytes=4, obytes=4)
    it_bytes = ab["bin"] + ab["blend_fwd"] + 1280 * 1024 * (12 + 4)
    hbm, hbm_src = peaks()
    it_gbs = it_bytes / (ms * 1e-3 / iters) / 1e9
    # CPU baseline: one iteration of the reference's steps on the oracle port
    # (render at the prior, Sobel selection, residual gate, pose rows, H^T R^-1 H)
    cpu = None
    if not args.no_cpu_baseline:
        from types import SimpleNamespace
        from scipy import ndimage
        from oracle import raster as orc
        f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
        P = {"means": f32(means), "rots": f32(rots), "scales": f32(scales), "opacities": f32(opac), "shs": f32(shs)}
        ost = SimpleNamespace(near=0.01, dilation=0.3, alpha_clamp=0.99, transmittance_min=1e-4, footprint_sigma=6.0,
                              alpha_cut=args.alpha_cut, max_footprint_px=512.0, background=np.zeros(3), sh_degree=0)
        obs = observed.cpu().numpy().astype(np.float64)
        t0 = time.perf_counter()
        T_cw = T_wc0.inverse()
        ref = orc.render(P, T_cw.R, T_cw.t, cam, ost)
        gray = obs.mean(axis=2)
        mag = np.hypot(ndimage.sobel(gray, axis=1, mode="nearest") / 8.0,
                       ndimage.sobel(gray, axis=0, mode="nearest") / 8.0)
        ids = np.flatnonzero((mag > fcfg.grad_threshold) & (ref["t_final"].reshape(1024, 1280) <
                                                            fcfg.coverage_max_transmittance))
        if len(ids) > fcfg.pixel_budget:
            ids = ids[np.unique(np.round(np.linspace(0, len(ids) - 1, fcfg.pixel_budget)).astype(int))]
        res = gray.reshape(-1)[ids] - ref["image"].reshape(-1, 3)[ids].mean(axis=1)
        keep = np.abs(res) <= fcfg.photo_gate
        H = -orc.pose_rows(ref, ids[keep], T_IC.R, T_IC.t)
        _ = H.T @ H, H.T @ res[keep]
        t_it = time.perf_counter() - t0
        cpu = {"value": 1.0 / t_it, "unit": "iterations/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"one IESKF iteration's measurement (render at the prior, selection, {int(keep.sum())} pose "
                         f"rows, H/b) on the oracle port ({t_it:.2f} s); the 15x15 algebra excluded"}
    if rank == 0:
        print(json.dumps({
            "metric": "IESKF photometric update iterations/s (config 4)", "value": iters / (ms * 1e-3),
            "unit": "iterations/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "replicas", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "roofline": {"bound": "hbm", "kernel": "one iteration (render + selection + pose rows + H/b)",
                         "achieved": it_gbs, "peak": hbm, "peak_source": hbm_src, "unit": "GB/s",
                         "frac": it_gbs / hbm, "algorithmic_bytes_per_iteration": it_bytes,
                         "traffic": (lambda t: None if t is None else t / iters)(
                             profile_figure("traffic.json", "cfg4", "unit")),
                         "traffic_note": AUX_TRAFFIC_NOTE + " per update / iterations",
                         "note": "host-synchronised filter iterations: latency bound, not bandwidth bound"},
            "cpu_baseline": cpu,
            "config": {"workload": "cfg4", "gaussians": len(means), "width": 1280, "height": 1024,
                       "iterations": iters, "alpha_cut": args.alpha_cut,
                       "timing": "host wall clock per full update (includes the per-iteration host syncs "
                                 "the filter needs)", "posterior_translation_error_m": err_t},
            "clocks": clk.summary(),
        }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="target", choices=sorted(CONFIGS) + ["cfg3", "cfg4", "window", "lidar"])
    ap.add_argument("--alpha-cut", type=float, default=1.0 / 255.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--lanes", type=int, default=8, help="concurrent view pipelines per GPU")
    ap.add_argument("--no-graph", dest="graph", action="store_false", help="eager launches instead of a CUDA graph")
    ap.add_argument("--copy-streams", type=int, default=1, help="H2D staging streams for the e2e pass")
    ap.add_argument("--frames", default="u8", choices=["u8", "f32"],
                    help="observed frames: 8-bit (the dataset's PPM frames, u/255 like read_ppm) or float32")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="N>1 gradient exchange: NCCL all-reduce + Adam, or the fused peer-memory step")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: run every rank on GPU 0 (exercises the N > 1 path on a
    # one-GPU box; with LSB_BENCH_BACKEND=gloo, since NCCL needs one GPU per rank)
    if os.environ.get("LSB_BENCH_SHARE_GPU") == "1":
        local_rank = 0
    if args.impl == "reference" and args.config in ("cfg3", "cfg4", "window", "lidar"):
        if rank == 0:
            print(json.dumps({"impl": "reference", "config": {"workload": args.config},
                              "unavailable": "the reference arm times the splat step (cfg1/cfg2/cfg5); this "
                                             "config's own line carries the oracle's cpu_baseline"}), flush=True)
        return
    if args.config == "cfg3":
        run_voxel(args, rank, world, local_rank)
        return
    if args.config == "cfg4":
        run_ieskf(args, rank, world, local_rank)
        return
    if args.config == "window":
        run_window(args, rank, world, local_rank)
        return
    if args.config == "lidar":
        run_lidar(args, rank, world, local_rank)
        return
    wl = build_workload(args.config, args.alpha_cut)
    if args.impl == "reference":
        run_reference(args, wl, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        backend = os.environ.get("LSB_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    run_ours(args, wl, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
