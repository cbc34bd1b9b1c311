"""Planner overrides (tdc_conv_plan_ex) and the measured autotune (NEXT-3)."""
import numpy as np
import pytest

import oracle
import synth
from synth import LayerShape
from paper_2211_03715_b200 import autotune


def test_coordinate_descent_finds_separable_optimum():
    knobs = {"a": [0, 1, 2, 3], "b": [0, 10, 20], "c": [0, 5]}
    target = {"a": 2, "b": 20, "c": 0}
    cost = lambda h: 1.0 + sum(abs(h[k] - target[k]) for k in knobs)
    r = autotune.coordinate_descent(cost, knobs)
    assert r.best_hints == target and r.best_us == 1.0
    assert r.planner_us == cost({"a": 0, "b": 0, "c": 0}) and r.gap > 0
    # determinism and the cache: a second run measures the same points
    assert autotune.coordinate_descent(cost, knobs).best_hints == target


def test_coordinate_descent_skips_invalid_points():
    knobs = {"a": [0, 1, 2]}
    r = autotune.coordinate_descent(lambda h: None if h["a"] == 1 else 5.0 - h["a"], knobs)
    assert r.best_hints == {"a": 2}
    with pytest.raises(ValueError):
        autotune.coordinate_descent(lambda h: None, knobs)


@pytest.mark.gpu
@pytest.mark.parametrize("hints", [
    {"core3": 0}, {"bn_core": 32}, {"bn_stage1": 32, "bn_stage3": 64}, {"core3": 0, "ksplit_core": 2},
    {"ksplit_stage1": 2, "core3": 0, "ksplit_stage3": 2}, {"bn_core": 128, "core3": 0},
], ids=lambda h: "_".join(f"{k}{v}" for k, v in h.items()))
def test_planner_overrides_parity(hints):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2211_03715_b200 import tdc
    s = LayerShape(2, 128, 128, 14, 13, 64, 64, 3, 1, 1)
    d = synth.make_layer(s, seed=4, bias=True)
    plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16, hints=hints)
    info = plan.info()
    if hints.get("core3") == 0:
        assert info.core3 == 0
    if "bn_core" in hints:
        assert info.bn_core <= hints["bn_core"]
    if "ksplit_core" in hints:
        assert info.ksplit_core == hints["ksplit_core"]
    x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
    y = torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda")
    plan.forward(x, y)
    torch.cuda.synchronize()
    plan.close()
    got = synth.nhwc_to_nchw(y.cpu().numpy()).astype(np.float64)
    ref = oracle.tkd_stages(d["x"], d["core"], d["u_in"], d["u_out"], d["bias"], s.stride, s.pad)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) <= 1e-4
