"""Parity gate on the exact configuration bench.py times (VERDICT r1 'next' 1a/1b):
the 16 Tucker-ResNet-18 3x3 TKD layers at batch 32, headline math (3xBF16), NHWC,
launched the way the bench launches them (one CUDA graph of the whole step,
replayed), checked bit for bit against plain stream launches and, on full images,
against the fp64 oracle (reading R13: max-normalized error <= 1e-4)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

B = 32
IMAGES = (0, 15, 31)


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2211_03715_b200 import tdc
    return torch, tdc


def bench_layers(tdc, torch, math):
    """The bench's step: (layer id, shape) in R18 order, each with its own seeded
    weights and input (the seed does not depend on the rank)."""
    out, lid = [], 0
    for shape, count in synth.R18_SHAPES:
        for _ in range(count):
            s = shape.with_batch(B)
            d = synth.make_layer(s, seed=synth.BASE_SEED, layer_id=lid)
            plan = tdc.ConvPlan(s, d, layout=tdc.TDC_LAYOUT_NHWC, math=tdc.MATH_NAMES[math])
            x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
            y = torch.full((B, s.Ho, s.Wo, s.N), float("nan"), device="cuda")
            out.append({"lid": lid, "s": s, "d": d, "plan": plan, "x": x, "y": y})
            lid += 1
    return out


def test_graph_replay_equals_plain_launches(env):
    torch, tdc = env
    layers = bench_layers(tdc, torch, "3xbf16")
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for L in layers:
            L["plan"].forward(L["x"], L["y"], stream=stream)
    torch.cuda.synchronize()
    ref = [L["y"].clone() for L in layers]
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        for L in layers:
            L["plan"].forward(L["x"], L["y"], stream=stream)
    for rep in range(3):
        for L in layers:
            L["y"].fill_(float("nan"))
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            graph.replay()
        torch.cuda.synchronize()
        for L, r in zip(layers, ref):
            assert torch.equal(L["y"], r), (rep, L["s"].name, L["lid"])
    del graph
    for L in layers:
        L["plan"].close()


@pytest.mark.parametrize("shape,count", synth.R18_SHAPES, ids=[s.name for s, _ in synth.R18_SHAPES])
def test_full_images_at_bench_batch(env, shape, count):
    """B = 32 forward in the bench's launch configuration; images 0, 15 and 31 compared
    element by element with the fp64 oracle."""
    torch, tdc = env
    s = shape.with_batch(B)
    d = synth.make_layer(s, seed=synth.BASE_SEED)
    plan = tdc.ConvPlan(s, d, layout=tdc.TDC_LAYOUT_NHWC, math=tdc.TDC_MATH_3XBF16)
    x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
    y = torch.full((B, s.Ho, s.Wo, s.N), float("nan"), device="cuda")
    plan.forward(x, y)
    torch.cuda.synchronize()
    info = plan.info()
    plan.close()
    assert "3xbf16" in info.variant_name, info.variant_name
    got = synth.nhwc_to_nchw(y.cpu().numpy())[list(IMAGES)].astype(np.float64)
    ref = oracle.tkd_stages(d["x"][list(IMAGES)], d["core"], d["u_in"], d["u_out"], None, s.stride, s.pad)
    e = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
    assert e <= 1e-4, (s.name, info.variant_name, e)
