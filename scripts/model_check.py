import sys, numpy as np
sys.path.insert(0, '.')
import synth.models as sm, oracle.model as om, torch
from paper_2211_03715_b200 import tdc
for depth, width, image in [(18, 16, 32), (50, 16, 32), (18, 64, 224), (50, 64, 224)]:
    ops = sm.tucker_resnet(depth, image=image, num_classes=1000 if width == 64 else 37, width=width, seed=7)
    x = sm.model_input(2, image, seed=7)
    m = tdc.Model(ops, 2)
    h, w, c = m.output_shape()
    xd = torch.from_numpy(x).cuda(); out = torch.full((2, h, w, c), float('nan'), device='cuda')
    m.forward(xd, out); torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.float64)
    ref = om.forward(ops, x)
    print(depth, width, image, "err", np.max(np.abs(got - ref)) / np.max(np.abs(ref)), "nan", np.isnan(got).sum(), flush=True)
    m.close()
