"""Debug: graph-replayed µs of the Tucker VGG-16 224x224 / 112x112 TKD layers (r = 3/8) at a
few batches, planner default vs an env override (A/B).  Usage: python scripts/vgg_layer_time.py"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from synth import LayerShape
from paper_2211_03715_b200 import tdc, roofline as rl
for base in [LayerShape(1, 64, 64, 224, 224, 24, 24, 3, 1, 1, "vgg_224_r3/8"),
             LayerShape(1, 128, 128, 112, 112, 48, 48, 3, 1, 1, "vgg_112_r3/8")] + synth.PAPER_WEAK_SHAPES:
    for B in (1, 8, 64):
        sh = base.with_batch(B)
        d = synth.make_layer(sh)
        p = tdc.ConvPlan(sh, d, math=tdc.TDC_MATH_3XBF16)
        x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
        y = torch.empty((sh.B, sh.Ho, sh.Wo, sh.N), device="cuda")
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for _ in range(3):
                p.forward(x, y, stream=st)
        g = torch.cuda.CUDAGraph()
        n = 10
        with torch.cuda.graph(g, stream=st):
            for _ in range(n):
                p.forward(x, y, stream=st)
        with torch.cuda.stream(st):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with torch.cuda.stream(st):
            for _ in range(3):
                g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (3 * n)
        gbs = rl.tkd_bytes(sh) / us / 1e3
        print(f"{base.name:28s} B={B:3d} {p.info().variant_name:22s} {us:9.2f} us {gbs:8.1f} GB/s", flush=True)
        del g
        p.close()
