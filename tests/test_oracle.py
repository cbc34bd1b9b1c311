"""Pins for the fp64 CPU oracle (oracle/), checked against things other than itself.

Each test names what fixes the expected value: a closed form from the paper /
SPEC (tests/golden/*.json, cited there), a library routine the oracle does not
use (torch fp64 conv2d, numpy matmul), an exact integer computation, a
scatter-form brute force with a different loop structure, or an invariant of
the method (Eq. tkd2).  A plausible mistake in the oracle -- a dropped
tap, a wrong sign or index, a transposed factor, a missing pad/stride term --
fails at least one of them.
"""
import itertools

import numpy as np
import pytest
import torch

import oracle
import synth
from synth import LayerShape


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


# ---------------------------------------------------------------- closed forms
def test_golden_valid_2x2_ones(golden):
    g = golden("spec_conv_examples.json")
    x = np.array(g["x"], dtype=np.float64)[None, None]
    case = g["valid_2x2_ones"]
    w = np.ones((1, 1, case["kernel"], case["kernel"]))
    y = oracle.conv7(x, w, case["stride"], case["pad"])
    assert np.array_equal(y[0, 0], np.array(case["y"], dtype=np.float64))


@pytest.mark.parametrize("case", ["same_3x3_ones", "stride2_3x3_ones"])
def test_golden_padded_ones(golden, case):
    g = golden("spec_conv_examples.json")
    x = np.array(g["x"], dtype=np.float64)[None, None]
    c = g[case]
    w = np.ones((1, 1, c["kernel"], c["kernel"]))
    y = oracle.conv7(x, w, c["stride"], c["pad"])
    assert np.array_equal(y[0, 0], np.array(c["y"], dtype=np.float64))


def test_golden_impulse_is_cross_correlation(golden):
    """Reading R4: cross-correlation, so the kernel appears flipped."""
    c = golden("spec_conv_examples.json")["impulse_ramp"]
    x = np.array(c["x"], dtype=np.float64)[None, None]
    w = np.array(c["w"], dtype=np.float64)[None, None]
    y = oracle.conv7(x, w, 1, 1)
    assert np.array_equal(y[0, 0], np.array(c["y"], dtype=np.float64))


def test_golden_reconstruct_2x2(golden):
    g = golden("reconstruct_2x2.json")
    core = np.array(g["core_qa"], dtype=np.float64)[:, :, None, None]
    w = oracle.reconstruct(core, np.array(g["u_in"], float), np.array(g["u_out"], float))
    assert np.array_equal(w[:, :, 0, 0], np.array(g["w_nc"], dtype=np.float64))


def test_reconstruct_zero_core_is_zero():
    rng = np.random.default_rng(0)
    w = oracle.reconstruct(np.zeros((3, 2, 3, 3)), rng.standard_normal((5, 2)),
                           rng.standard_normal((4, 3)))
    assert w.shape == (4, 5, 3, 3) and not np.any(w)


def test_reconstruct_rank1_outer_product():
    """D1 = D2 = 1: W[n,c,r,t] = u_out[n] * g[r,t] * u_in[c] (separable kernel)."""
    rng = np.random.default_rng(1)
    ui, uo, g = rng.standard_normal((6, 1)), rng.standard_normal((5, 1)), rng.standard_normal((3, 3))
    w = oracle.reconstruct(g[None, None], ui, uo)
    for n in range(5):
        for c in range(6):
            np.testing.assert_allclose(w[n, c], uo[n, 0] * g * ui[c, 0], rtol=1e-15, atol=0)


# ------------------------------------------------------------ library routines
CONV_CASES = [
    # B, C, N, H, W, R, S, stride, pad
    (1, 1, 1, 5, 5, 3, 3, 1, 1),
    (2, 3, 4, 7, 6, 3, 3, 1, 1),
    (2, 3, 4, 7, 6, 3, 3, 2, 1),
    (1, 4, 2, 9, 9, 5, 5, 2, 2),
    (3, 2, 3, 8, 5, 1, 1, 1, 0),
    (1, 5, 3, 6, 7, 3, 1, 1, 0),
    (1, 2, 2, 4, 4, 3, 3, 3, 0),
    (2, 6, 5, 11, 10, 3, 3, 2, 0),
]


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv7_matches_torch_fp64(case):
    B, C, N, H, W, R, S, s, p = case
    rng = np.random.default_rng(hash(case) % 2**32)
    x = rng.standard_normal((B, C, H, W))
    w = rng.standard_normal((N, C, R, S))
    y = oracle.conv7(x, w, s, p)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x), torch.from_numpy(w),
                                     stride=s, padding=p).numpy()
    assert y.shape == ref.shape
    assert _rel(y, ref) < 1e-13


def test_stage1_and_stage3_match_numpy_matmul():
    """Stages 1 and 3 are 1x1 convs: a matrix product per pixel (SURVEY §8(c) pin 1)."""
    s = LayerShape(2, 12, 10, 9, 7, 5, 6, 3, 2, 1)
    d = synth.make_layer(s, seed=3)
    y, x1, z = oracle.tkd_stages(d["x"], d["core"], d["u_in"], d["u_out"], None,
                                 s.stride, s.pad, return_intermediates=True)
    x64 = d["x"].astype(np.float64)
    x1_ref = np.matmul(x64.transpose(0, 2, 3, 1).reshape(-1, s.C),
                       d["u_in"].astype(np.float64))
    x1_ref = x1_ref.reshape(s.B, s.H, s.W, s.D1).transpose(0, 3, 1, 2)
    assert _rel(x1, x1_ref) < 1e-13
    y_ref = np.matmul(z.transpose(0, 2, 3, 1).reshape(-1, s.D2),
                      d["u_out"].astype(np.float64).T)
    y_ref = y_ref.reshape(s.B, s.Ho, s.Wo, s.N).transpose(0, 3, 1, 2)
    assert _rel(y, y_ref) < 1e-13
    # stage 2 alone against torch
    z_ref = torch.nn.functional.conv2d(torch.from_numpy(x1), torch.from_numpy(
        d["core"].astype(np.float64)), stride=s.stride, padding=s.pad).numpy()
    assert _rel(z, z_ref) < 1e-13


# ------------------------------------------------------------ method invariants
@pytest.mark.parametrize("shape", [
    synth.CONFIG1,
    LayerShape(2, 16, 24, 10, 9, 8, 6, 3, 2, 1),
    LayerShape(1, 8, 8, 6, 6, 3, 5, 5, 1, 2),
    LayerShape(1, 9, 7, 5, 8, 2, 3, 1, 1, 0),
    LayerShape(2, 6, 6, 7, 7, 4, 4, 3, 1, 0),
])
def test_three_stage_equals_reconstructed_kernel(shape):
    """P:L693 Eq. tkd2 + linearity: three stages == one conv with W_rec."""
    d = synth.make_layer(shape, seed=11, bias=True)
    y = oracle.tkd_stages(d["x"], d["core"], d["u_in"], d["u_out"], d["bias"],
                          shape.stride, shape.pad)
    y_full = oracle.tkd_full(d["x"], d["core"], d["u_in"], d["u_out"], d["bias"],
                             shape.stride, shape.pad)
    assert y.shape == (shape.B, shape.N, shape.Ho, shape.Wo)
    assert _rel(y, y_full) < 1e-12


@pytest.mark.parametrize("stride,pad", [(1, 1), (2, 1), (1, 0)])
def test_identity_factors_full_rank_is_plain_conv(stride, pad):
    """D1=C, D2=N, U=I: the TKD layer is bit-identical to conv7(x, core) (north_star)."""
    C, N = 5, 4
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, C, 7, 6))
    core = rng.standard_normal((N, C, 3, 3))
    y = oracle.tkd_stages(x, core, np.eye(C), np.eye(N), None, stride, pad)
    assert np.array_equal(y, oracle.conv7(x, core, stride, pad))


def test_linearity():
    s = LayerShape(1, 6, 5, 6, 6, 3, 2, 3, 1, 1)
    d = synth.make_layer(s, seed=2)
    rng = np.random.default_rng(9)
    x2 = rng.standard_normal(d["x"].shape)
    f = lambda x: oracle.tkd_stages(x, d["core"], d["u_in"], d["u_out"], None, 1, 1)
    lhs = f(2.5 * d["x"].astype(np.float64) - 0.75 * x2)
    rhs = 2.5 * f(d["x"]) - 0.75 * f(x2)
    assert _rel(lhs, rhs) < 1e-12


def test_integer_inputs_are_exact():
    """Integer tensors: the fp64 oracle must equal an exact int64 evaluation."""
    s = LayerShape(2, 16, 16, 8, 8, 4, 4, 3, 1, 1)
    d = synth.make_layer(s, seed=42, integer=True, bias=True)
    xi = d["x"].astype(np.int64)
    x1 = np.einsum("bchw,ca->bahw", xi, d["u_in"].astype(np.int64))
    xp = np.pad(x1, ((0, 0), (0, 0), (1, 1), (1, 1)))
    z = np.zeros((s.B, s.D2, s.Ho, s.Wo), dtype=np.int64)
    g = d["core"].astype(np.int64)
    for r in range(3):
        for t in range(3):
            z += np.einsum("bahw,qa->bqhw", xp[:, :, r:r + s.Ho, t:t + s.Wo], g[:, :, r, t])
    y_int = np.einsum("bqhw,nq->bnhw", z, d["u_out"].astype(np.int64)) \
        + d["bias"].astype(np.int64)[None, :, None, None]
    y = oracle.tkd_stages(d["x"], d["core"], d["u_in"], d["u_out"], d["bias"], 1, 1)
    assert np.array_equal(y, y_int.astype(np.float64))
    assert np.max(np.abs(y_int)) < 2 ** 24


# ---------------------------------------------------------- scatter brute force
def _scatter_tkd(x, core, u_in, u_out, stride, pad):
    """Scatter form: every input element pushes its contributions forward.
    Different loop structure from the oracle's gather loops."""
    B, C, H, W = x.shape
    D2, D1, K, _ = core.shape
    N = u_out.shape[0]
    Ho, Wo = (H + 2 * pad - K) // stride + 1, (W + 2 * pad - K) // stride + 1
    x1 = np.zeros((B, D1, H, W))
    for b, c, h, w in itertools.product(range(B), range(C), range(H), range(W)):
        for a in range(D1):
            x1[b, a, h, w] += x[b, c, h, w] * u_in[c, a]
    z = np.zeros((B, D2, Ho, Wo))
    for b, a, h, w in itertools.product(range(B), range(D1), range(H), range(W)):
        for r, t in itertools.product(range(K), range(K)):
            ni, nj = h + pad - r, w + pad - t
            if ni % stride or nj % stride:
                continue
            i, j = ni // stride, nj // stride
            if 0 <= i < Ho and 0 <= j < Wo:
                for q in range(D2):
                    z[b, q, i, j] += x1[b, a, h, w] * core[q, a, r, t]
    y = np.zeros((B, N, Ho, Wo))
    for b, q, i, j in itertools.product(range(B), range(D2), range(Ho), range(Wo)):
        for n in range(N):
            y[b, n, i, j] += z[b, q, i, j] * u_out[n, q]
    return y


TINY = [c for c in itertools.product((1, 3), (1, 2), (1, 2), (1, 2), (1, 3, 5), (2, 5),
                                     (1, 3), (1, 2), (0, 1))
        if c[6] <= min(c[4], c[5]) + 2 * c[8]]


def test_tiny_layers_match_scatter_brute_force():
    rng = np.random.default_rng(123)
    for (C, N, D1, D2, H, W, K, s, p) in TINY:
        x = rng.standard_normal((1, C, H, W))
        core = rng.standard_normal((D2, D1, K, K))
        ui, uo = rng.standard_normal((C, D1)), rng.standard_normal((N, D2))
        y = oracle.tkd_stages(x, core, ui, uo, None, s, p)
        ref = _scatter_tkd(x, core, ui, uo, s, p)
        assert y.shape == ref.shape
        assert np.max(np.abs(y - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref))), (C, N, D1, D2, H, W, K, s, p)


def test_operator_columns_are_impulse_responses():
    """Dense operator M by scatter; column k must equal oracle(e_k) exactly-ish."""
    C, N, D1, D2, H, W, K, s, p = 2, 2, 2, 1, 4, 3, 3, 2, 1
    rng = np.random.default_rng(7)
    core = rng.standard_normal((D2, D1, K, K))
    ui, uo = rng.standard_normal((C, D1)), rng.standard_normal((N, D2))
    for k in range(C * H * W):
        e = np.zeros(C * H * W)
        e[k] = 1.0
        e = e.reshape(1, C, H, W)
        col = _scatter_tkd(e, core, ui, uo, s, p)
        np.testing.assert_allclose(oracle.tkd_stages(e, core, ui, uo, None, s, p), col,
                                   rtol=1e-13, atol=1e-13)


# --------------------------------------------------------- sampled point eval
@pytest.mark.parametrize("shape", [
    LayerShape(2, 16, 12, 9, 10, 6, 5, 3, 1, 1),
    LayerShape(2, 16, 12, 9, 10, 6, 5, 3, 2, 1),
    LayerShape(1, 5, 7, 6, 4, 3, 2, 5, 1, 2),
])
def test_point_eval_bit_identical_to_stages(shape):
    d = synth.make_layer(shape, seed=4, bias=True)
    y = oracle.tkd_stages(d["x"], d["core"], d["u_in"], d["u_out"], d["bias"],
                          shape.stride, shape.pad)
    pts = synth.sample_points(shape, 40)
    v = oracle.tkd_points(d["x"], d["core"], d["u_in"], d["u_out"], pts, d["bias"],
                          shape.stride, shape.pad)
    assert np.array_equal(v, np.array([y[p] for p in pts]))


def test_thread_count_does_not_change_bits():
    s = LayerShape(3, 8, 8, 10, 10, 4, 4, 3, 1, 1)
    d = synth.make_layer(s, seed=8)
    oracle.set_threads(1)
    a = oracle.tkd_stages(d["x"], d["core"], d["u_in"], d["u_out"], None, 1, 1)
    oracle.set_threads(4)
    b = oracle.tkd_stages(d["x"], d["core"], d["u_in"], d["u_out"], None, 1, 1)
    oracle.set_threads(0)
    assert np.array_equal(a, b)


def test_invalid_arguments_raise():
    with pytest.raises(ValueError):
        oracle.conv7(np.zeros((1, 1, 2, 2)), np.zeros((1, 1, 5, 5)), 1, 0)  # K > H + 2p
    with pytest.raises(ValueError):
        oracle.tkd_stages(np.zeros((1, 3, 4, 4)), np.zeros((2, 2, 3, 3)),
                          np.zeros((4, 2)), np.zeros((3, 2)))  # u_in rows != C
    assert oracle.out_dim(56, 3, 2, 1) == 28 and oracle.out_dim(7, 3, 1, 1) == 7
    assert oracle.out_dim(4, 3, 0, 0) < 0
