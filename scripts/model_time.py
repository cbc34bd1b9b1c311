"""Debug: ms per Tucker ResNet-50 / VGG-16 forward (CUDA graph replay)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth.models as sm
from paper_2211_03715_b200 import tdc
for arch, b in (("r50", 32), ("vgg16", 64)):
    ops = sm.tucker_resnet(50) if arch == "r50" else sm.tucker_vgg16()
    m = tdc.Model(ops, b)
    h, w, c = m.output_shape()
    x = torch.from_numpy(sm.model_input(b)).cuda()
    o = torch.empty((b, h, w, c), device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            m.forward(x, o, stream=st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        m.forward(x, o, stream=st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(20):
            g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    print(arch, round(e0.elapsed_time(e1) / 20, 3), "ms", os.environ.get("TDC_GEMM_DBG", "0"))
    m.close()
