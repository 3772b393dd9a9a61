import sys, torch, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from golden_io import load
from paper_2501_08672_b200.dist import adam_peer_step, shard_range
from paper_2501_08672_b200.optimize import AdamState, OptimConfig
from paper_2501_08672_b200.raster import GaussianArrays, ParamGradients
s = load("scene_room_0323")
base = GaussianArrays(s["means"], s["rots"], s["scales"], s["opacities"], s["shs"]).clone(torch.float64)
n, k = len(base), 1
g = torch.randn(n * 13, device="cuda") * 1e-3
cfg = OptimConfig()
for steps in (1, 2):
    ref = base.clone(); st = AdamState(ref, cfg)
    rep = [base.clone()]; t = [torch.zeros(n, dtype=torch.uint8, device="cuda")]; sp = AdamState(rep[0], cfg)
    for _ in range(steps):
        st.apply_dev(ref, ParamGradients.from_flat(g, n, k))
        adam_peer_step(rep, [g], t, 0, 0, n, sp)
    torch.cuda.synchronize()
    for name, a, b in (("m", sp.m, st.m), ("v", sp.v, st.v), ("scales", rep[0].scales.flatten(), ref.scales.flatten())):
        bad = (a != b).nonzero().flatten()
        print(steps, name, bad.numel(), bad[:4].tolist(), a[bad[:2]].tolist(), b[bad[:2]].tolist())
ref = base.clone(); st = AdamState(ref, cfg)
rep = [base.clone()]; t = [torch.zeros(n, dtype=torch.uint8, device="cuda")]; sp = AdamState(rep[0], cfg)
st.apply_dev(ref, ParamGradients.from_flat(g, n, k))
adam_peer_step(rep, [g], t, 0, 0, n, sp)
torch.cuda.synchronize()
s0 = float(base.scales[0, 0]); g0 = float(g[6 * n]); s1 = float(ref.scales[0, 0])
print("expect old-s", 0.1 * g0 * s0, "expect new-s", 0.1 * g0 * s1, "ref m", float(st.m[6 * n]), "peer m", float(sp.m[6 * n]))
