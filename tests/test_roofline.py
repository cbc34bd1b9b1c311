"""Pins of the bench's algorithmic-work numerators (roofline.py) -- the headline's
GB/s and TFLOP/s divide these, so they are checked against the SPEC worked example
(S:L438-444), a hand count, and an independent element count of the synthetic
tensors the bench actually allocates."""
import numpy as np

import synth
from paper_2211_03715_b200 import roofline as rl
from synth import LayerShape


def test_flops_match_spec_worked_example(golden):
    g = golden("flops_spec.json")  # H=W=14, C=N=256, 3x3, d1=d2=64
    s = LayerShape(1, g["C"], g["N"], g["H"], g["W"], g["D1"], g["D2"], g["K"], g["stride"], g["pad"])
    assert rl.stage_flops(s.H, s.W, s.C, s.N, s.D1, s.D2, s.K, s.stride, s.pad) == \
        (g["stage1"], g["stage2"], g["stage3"])
    assert rl.tkd_flops(s) == g["tucker"]
    assert rl.dense_flops(s) == g["orig"]


def test_bytes_hand_count_r18_56():
    # 56x56x64 -> 64, D = 32, B = 32 (the bench's dominant layer), counted by hand:
    # x: 32*56*56*64 floats, y: 32*56*56*64 floats, weights 64*32 + 32*32*9 + 32*64 floats
    s = LayerShape(32, 64, 64, 56, 56, 32, 32, 3, 1, 1)
    x = 32 * 56 * 56 * 64
    y = 32 * 56 * 56 * 64
    w = 64 * 32 + 32 * 32 * 9 + 32 * 64
    assert 4 * (x + y + w) == 51_433_472
    assert rl.tkd_bytes(s) == 51_433_472
    # FLOPs by hand: 2*B*(HWC*D1 + H'W'*D1*D2*9 + H'W'*D2*N)
    assert rl.tkd_flops(s) == 2 * 32 * (3136 * 64 * 32 + 3136 * 32 * 32 * 9 + 3136 * 32 * 64)


def test_bytes_equal_the_allocated_synthetic_tensors():
    """Second route: the byte count of the very arrays make_layer returns (x, core, U_in,
    U_out) plus an output of the oracle's shape, for every R18 shape and strides 1-2."""
    for shape, _ in synth.R18_SHAPES:
        s = shape.with_batch(2)
        d = synth.make_layer(s)
        y_elems = s.B * s.N * s.Ho * s.Wo
        nbytes = sum(np.asarray(d[k], dtype=np.float32).nbytes for k in ("x", "core", "u_in", "u_out")) + 4 * y_elems
        assert rl.tkd_bytes(s) == nbytes, s.name
        assert rl.tkd_bytes(s, bias=True) == nbytes + 4 * s.N


def test_paper_volumes_match_spec_worked_example(golden):
    g = golden("paper_model_spec.json")["volumes"]  # S:L250, Eqs. (3)-(6)
    s = LayerShape(1, 256, 256, g["H"], g["W"], g["C"], g["N"], g["R"], 1, 1)  # core sees D1=C, D2=N
    vk, vx, vy, tot = rl.paper_volumes(s, g["TH"], g["TW"], g["TC"])
    assert (vk, vx, vy, tot) == (g["vk"], g["vx"], g["vy"], g["total"])
    # single-tile reduction
    vk, vx, vy, _ = rl.paper_volumes(s, g["H"], g["W"], g["C"])
    assert vk == g["C"] * g["N"] and vx == g["C"] * (g["H"] + 2) * (g["W"] + 2) and vy == g["H"] * g["W"] * g["N"]
