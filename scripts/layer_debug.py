"""Debug of the single-launch layer kernel: structured weights isolate the stages."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
from synth import LayerShape
from paper_2211_03715_b200 import tdc


def run(s, d):
    plan = tdc.ConvPlan(s, d, layout=tdc.TDC_LAYOUT_NHWC, math=tdc.TDC_MATH_3XBF16)
    x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
    y = torch.full((s.B, s.Ho, s.Wo, s.N), float("nan"), device="cuda")
    plan.forward(x, y)
    torch.cuda.synchronize()
    name = plan.info().variant_name
    plan.close()
    return synth.nhwc_to_nchw(y.cpu().numpy()).astype(np.float64), name


def report(tag, s, d):
    got, name = run(s, d)
    ref = oracle.tkd_stages(d["x"], d["core"], d["u_in"], d["u_out"], None, s.stride, s.pad)
    bad = ~np.isclose(got, ref, atol=1e-3 * np.abs(ref).max())
    print(f"== {tag} {name}: max-norm err {np.nanmax(np.abs(got-ref))/np.abs(ref).max():.3e}, bad {bad.sum()}/{bad.size}, nan {np.isnan(got).sum()}")
    if bad.any():
        idx = np.argwhere(bad)
        print("   bad (b,n,i,j) first:", idx[:8].tolist())
        rows = np.unique(idx[:, 2]); cols = np.unique(idx[:, 3]); chans = np.unique(idx[:, 1])
        print("   bad rows", rows[:40].tolist(), "cols", cols[:40].tolist(), "chans", chans[:20].tolist(), len(chans))
        b, n, i, j = idx[0]
        print("   got", got[b, n, i, max(0,j-2):j+3], "ref", ref[b, n, i, max(0,j-2):j+3])


def ident(n):
    return np.eye(n, dtype=np.float32)


C = 32
for (H, W, K, B) in [(8, 8, 1, 1), (8, 8, 3, 1), (12, 10, 3, 2), (56, 56, 3, 1)]:
    s = LayerShape(B, C, C, H, W, C, C, K, 1, (K - 1) // 2)
    x = np.random.default_rng(0).integers(-3, 4, (B, C, H, W)).astype(np.float32)
    core = np.zeros((C, C, K, K), np.float32)
    for q in range(C):
        core[q, q, K // 2, K // 2] = 1.0
    d = {"x": x, "core": core, "u_in": ident(C), "u_out": ident(C), "bias": None}
    report(f"identity all, H{H} W{W} K{K} B{B}", s, d)
    d2 = dict(d)
    d2["u_in"] = np.random.default_rng(1).integers(-2, 3, (C, C)).astype(np.float32)
    report(f"random U_in, H{H} W{W} K{K}", s, d2)
    d3 = dict(d)
    d3["u_out"] = np.random.default_rng(2).integers(-2, 3, (C, C)).astype(np.float32)
    report(f"random U_out, H{H} W{W} K{K}", s, d3)
    if K == 3:
        for tap in [(0, 0), (2, 2), (0, 2)]:
            d4 = dict(d)
            c4 = np.zeros_like(core)
            for q in range(C):
                c4[q, q, tap[0], tap[1]] = 1.0
            d4["core"] = c4
            report(f"delta core at tap {tap}, H{H} W{W}", s, d4)
