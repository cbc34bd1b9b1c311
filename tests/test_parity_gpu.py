"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle.

Error metric (reading R13): max_i |y_i - y_ref_i| / max_i |y_ref_i|.
Tolerances (north_star): 1e-4 for FP32 and 3xTF32 math, 1e-2 for TF32.
Integer-valued layers (every partial sum an integer < 2^24) must be bit-exact
in FP32 math whatever the reduction order.
"""
import numpy as np
import pytest

import oracle
import synth
from synth import LayerShape

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "3xtf32": 1e-4, "3xbf16": 1e-4, "tf32": 1e-2}


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2211_03715_b200 import tdc
    return torch, tdc


def run_layer(env, shape, d, layout="nhwc", math="fp32", batch=None):
    torch, tdc = env
    lay = tdc.TDC_LAYOUT_NHWC if layout == "nhwc" else tdc.TDC_LAYOUT_NCHW
    plan = tdc.ConvPlan(shape, d, layout=lay, math=tdc.MATH_NAMES[math])
    b = shape.B if batch is None else batch
    x_np = d["x"][:b]
    if layout == "nhwc":
        x = torch.from_numpy(synth.nchw_to_nhwc(x_np)).cuda()
        y = torch.full((b, shape.Ho, shape.Wo, shape.N), float("nan"), device="cuda")
    else:
        x = torch.from_numpy(np.ascontiguousarray(x_np)).cuda()
        y = torch.full((b, shape.N, shape.Ho, shape.Wo), float("nan"), device="cuda")
    plan.forward(x, y, batch=b)
    torch.cuda.synchronize()
    out = y.cpu().numpy()
    info = plan.info()
    plan.close()
    if layout == "nhwc":
        out = synth.nhwc_to_nchw(out)
    return out, info


def err(got, ref):
    return float(np.max(np.abs(got.astype(np.float64) - ref)) / np.max(np.abs(ref)))


def ref_of(shape, d, b=None):
    x = d["x"] if b is None else d["x"][:b]
    return oracle.tkd_stages(x, d["core"], d["u_in"], d["u_out"], d["bias"], shape.stride, shape.pad)


MATHS = ["fp32", "tf32", "3xtf32", "3xbf16"]


@pytest.mark.parametrize("math", MATHS)
@pytest.mark.parametrize("layout", ["nhwc", "nchw"])
def test_config1(env, layout, math):
    s = synth.CONFIG1
    d = synth.make_layer(s)
    got, _ = run_layer(env, s, d, layout, math)
    assert np.all(np.isfinite(got))
    assert err(got, ref_of(s, d)) <= TOL[math]


@pytest.mark.parametrize("math", ["fp32", "3xtf32", "3xbf16"])
@pytest.mark.parametrize("layout", ["nhwc", "nchw"])
def test_integer_layer_is_bit_exact(env, layout, math):
    """Every partial sum is an integer < 2^16: fp32 FFMA and the exact hi/lo splits
    (3xTF32, 3xBF16: hi + lo == value) must reproduce the oracle bit for bit."""
    s = LayerShape(2, 16, 16, 8, 8, 4, 4, 3, 1, 1)
    d = synth.make_layer(s, integer=True, bias=True)
    got, _ = run_layer(env, s, d, layout, math)
    assert np.array_equal(got.astype(np.float64), ref_of(s, d))


@pytest.mark.parametrize("shape", [
    LayerShape(3, 37, 29, 13, 11, 7, 5, 3, 1, 1),     # ragged C, N, D, H, W
    LayerShape(2, 33, 18, 15, 9, 6, 3, 3, 2, 1),      # stride 2, odd sizes
    LayerShape(1, 8, 12, 10, 10, 3, 5, 5, 1, 2),      # 5x5 core
    LayerShape(2, 12, 8, 9, 7, 4, 4, 1, 1, 0),        # 1x1 core
    LayerShape(1, 16, 16, 9, 9, 4, 4, 3, 3, 0),       # stride 3, no pad
    LayerShape(1, 5, 3, 3, 3, 2, 2, 3, 1, 1),         # smaller than a tile
    LayerShape(1, 64, 64, 1, 1, 16, 16, 3, 1, 1),     # 1x1 image, all padding
    LayerShape(2, 64, 96, 20, 17, 64, 96, 3, 1, 1),   # full ranks
    LayerShape(1, 8, 8, 30, 30, 4, 4, 3, 24, 1),      # stride 24 > K*K phases
    LayerShape(1, 8, 8, 20, 20, 4, 4, 7, 8, 3),       # 7x7 core, stride 8
])
@pytest.mark.parametrize("math", MATHS)
def test_ragged_and_edge_shapes(env, shape, math):
    d = synth.make_layer(shape, seed=7, bias=True)
    got, info = run_layer(env, shape, d, "nhwc", math)
    # the variant that ran is asserted, so no case silently exercises another kernel:
    # TMA needs 16-byte pixel rows (C % 4 == 0); otherwise every mode uses the FP32 kernel
    if shape.C % 4:
        assert info.variant_name == "fused_simt_fp32", info.variant_name
    elif math == "fp32":  # CUDA-core three-launch GEMM-with-taps path (s*s phases <= 49)
        assert info.variant_name == ("simt3_fp32" if shape.stride ** 2 <= 49 else "fused_simt_fp32"), \
            info.variant_name
    elif math == "3xbf16":  # fp32-grade split; 3xTF32 where the 3xBF16 band does not fit (stride 3: 9 phases)
        assert "3xbf16" in info.variant_name or "3xtf32" in info.variant_name, info.variant_name
    else:
        assert info.variant_name != "fused_simt_fp32", info.variant_name
    assert err(got, ref_of(shape, d)) <= TOL[math]


@pytest.mark.parametrize("shape,count", synth.R18_SHAPES, ids=[s.name for s, _ in synth.R18_SHAPES])
@pytest.mark.parametrize("math", MATHS)
def test_r18_shapes_batch1_full(env, shape, count, math):
    d = synth.make_layer(shape, seed=synth.BASE_SEED)
    got, _ = run_layer(env, shape, d, "nhwc", math)
    assert err(got, ref_of(shape, d)) <= TOL[math]


@pytest.mark.parametrize("shape,count", synth.R18_SHAPES, ids=[s.name for s, _ in synth.R18_SHAPES])
@pytest.mark.parametrize("math", MATHS)
def test_r18_shapes_batch32_sampled(env, shape, count, math):
    """Full benchmark size (B=32, the bench's launch configuration), checked on
    sampled outputs the oracle evaluates one by one."""
    s = shape.with_batch(32)
    d = synth.make_layer(s, seed=synth.BASE_SEED)
    got, _ = run_layer(env, s, d, "nhwc", math)
    assert np.all(np.isfinite(got))
    pts = synth.sample_points(s, 200)
    ref = oracle.tkd_points(d["x"], d["core"], d["u_in"], d["u_out"], pts, None, s.stride, s.pad)
    vals = np.array([got[p] for p in pts], dtype=np.float64)
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(vals - ref)) / scale <= TOL[math]


@pytest.mark.parametrize("shape,count", synth.R18_SHAPES, ids=[s.name for s, _ in synth.R18_SHAPES])
def test_fp32_variant_is_the_cuda_core_gemm(env, shape, count):
    torch, tdc = env
    plan = tdc.ConvPlan(shape.with_batch(32), synth.make_layer(shape), math=tdc.TDC_MATH_FP32)
    assert plan.info().variant_name == "simt3_fp32" and plan.info().launches_per_forward == 3
    plan.close()


def test_fp32_old_single_kernel_path_still_matches(env, monkeypatch):
    """TDC_NO_SGEMM keeps the single-kernel SIMT variant reachable (C % 4 != 0 uses it)."""
    monkeypatch.setenv("TDC_NO_SGEMM", "1")
    s = LayerShape(2, 32, 24, 10, 9, 8, 12, 3, 2, 1)
    d = synth.make_layer(s, seed=3, bias=True)
    got, info = run_layer(env, s, d, "nhwc", "fp32")
    assert info.variant_name == "fused_simt_fp32"
    assert err(got, ref_of(s, d)) <= TOL["fp32"]


@pytest.mark.parametrize("shape,count", synth.R18_SHAPES, ids=[s.name for s, _ in synth.R18_SHAPES])
def test_tensor_core_variant_is_selected(env, shape, count):
    torch, tdc = env
    d = synth.make_layer(shape)
    plan = tdc.ConvPlan(shape.with_batch(32), d, math=tdc.TDC_MATH_TF32)
    assert plan.info().variant_name in ("fused_tc_tf32", "tc3_tf32_band", "tc3_tf32")
    plan.close()


@pytest.mark.parametrize("shape", [s for s, _ in synth.R18_SHAPES] + [
    LayerShape(3, 64, 40, 13, 11, 24, 20, 3, 1, 1),
    LayerShape(2, 32, 48, 15, 9, 16, 32, 3, 2, 1),
], ids=lambda s: s.name or f"{s.C}_{s.N}_{s.H}x{s.W}_s{s.stride}")
def test_three_launch_tensor_core_path(env, shape, monkeypatch):
    """The unfused tcgen05 path (forced with TDC_DISABLE_FUSED) on its own."""
    monkeypatch.setenv("TDC_DISABLE_FUSED", "1")
    d = synth.make_layer(shape.with_batch(2), seed=13, bias=True)
    got, info = run_layer(env, shape.with_batch(2), d, "nhwc", "tf32")
    assert info.variant_name.startswith("tc3")
    assert err(got, ref_of(shape.with_batch(2), d)) <= TOL["tf32"]


@pytest.mark.parametrize("math", MATHS)
def test_partial_batch_and_batch_independence(env, math):
    s = LayerShape(8, 32, 32, 14, 14, 16, 16, 3, 1, 1)
    d = synth.make_layer(s, seed=3)
    full, _ = run_layer(env, s, d, math=math)
    part, _ = run_layer(env, s, d, batch=3, math=math)
    one, _ = run_layer(env, s.with_batch(1), {**d, "x": d["x"][:1]}, math=math)
    assert np.array_equal(part, full[:3])
    assert np.array_equal(one[0], full[0])


@pytest.mark.parametrize("math", MATHS)
def test_deterministic(env, math):
    s = LayerShape(4, 64, 64, 28, 28, 32, 32, 3, 1, 1)
    d = synth.make_layer(s, seed=5)
    a, _ = run_layer(env, s, d, math=math)
    b, _ = run_layer(env, s, d, math=math)
    assert np.array_equal(a, b)


def test_forward_host_matches_device(env):
    torch, tdc = env
    s = LayerShape(4, 32, 48, 12, 12, 8, 12, 3, 2, 1)
    d = synth.make_layer(s, seed=9, bias=True)
    plan = tdc.ConvPlan(s, d, layout=tdc.TDC_LAYOUT_NHWC)
    xh = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).pin_memory()
    yh = torch.empty((s.B, s.Ho, s.Wo, s.N)).pin_memory()
    plan.forward_host(xh, yh)
    dev, _ = run_layer(env, s, d)
    assert np.array_equal(synth.nhwc_to_nchw(yh.numpy()), dev)
    plan.close()


def test_forward_rejects_bad_calls(env):
    torch, tdc = env
    s = synth.CONFIG1
    d = synth.make_layer(s)
    plan = tdc.ConvPlan(s, d)
    x = torch.zeros((1, 8, 8, 16), device="cuda")
    with pytest.raises(tdc.TdcError):
        plan.forward(x, x)  # aliasing
    y = torch.zeros((2, 8, 8, 16), device="cuda")
    with pytest.raises(tdc.TdcError):
        tdc.tdc_conv_forward(plan._h, x.data_ptr(), y.data_ptr(), 2)  # batch > plan
    plan.close()


@pytest.mark.parametrize("fuse3", [True, False], ids=["core3", "three_launch"])
@pytest.mark.parametrize("shape", [s for s, _ in synth.R18_SHAPES] + [
    LayerShape(3, 64, 40, 13, 11, 24, 20, 3, 1, 1),
    LayerShape(2, 32, 48, 15, 9, 16, 32, 3, 2, 1),
    LayerShape(2, 40, 72, 12, 10, 40, 48, 5, 1, 2),
    # small M, long K: split-K over clusters (stages 1 and 3)
    LayerShape(2, 512, 256, 5, 7, 256, 128, 3, 1, 1),
    LayerShape(3, 256, 512, 4, 4, 128, 256, 3, 2, 1),
    LayerShape(1, 320, 96, 3, 3, 192, 64, 1, 1, 0),
], ids=lambda s: s.name or f"{s.C}_{s.N}_{s.H}x{s.W}_k{s.K}_s{s.stride}")
def test_3xbf16_core3_and_three_launch(env, shape, fuse3, monkeypatch):
    """3xBF16 with stage 3 fused into the core kernel (Z on chip) where it fits,
    and the three-launch path forced with TDC_NO_FUSE3, against the oracle."""
    if not fuse3:
        monkeypatch.setenv("TDC_NO_FUSE3", "1")
    s = shape.with_batch(2)
    d = synth.make_layer(s, seed=21, bias=True)
    got, info = run_layer(env, s, d, "nhwc", "3xbf16")
    assert "3xbf16" in info.variant_name, info.variant_name
    if not fuse3:
        assert info.variant_name in ("tc3_3xbf16_band", "tc3_3xbf16_pair")
    assert err(got, ref_of(s, d)) <= TOL["3xbf16"]


@pytest.mark.parametrize("shape,count", synth.R18_SHAPES, ids=[s.name for s, _ in synth.R18_SHAPES])
def test_3xbf16_variant_names(env, shape, count):
    torch, tdc = env
    d = synth.make_layer(shape)
    plan = tdc.ConvPlan(shape.with_batch(32), d, math=tdc.TDC_MATH_3XBF16)
    info = plan.info()
    assert info.variant_name in ("layer_3xbf16_fused", "tc2_3xbf16_core3", "tc3_3xbf16_band", "tc3_3xbf16_pair")
    assert info.launches_per_forward == {"layer_3xbf16_fused": 1, "tc2_3xbf16_core3": 2,
                                         "tc3_3xbf16_band": 3, "tc3_3xbf16_pair": 3}[info.variant_name]
    assert 0 < info.smem_bytes_per_cta <= 227 * 1024  # the reported footprint of the kernel that runs
    plan.close()


@pytest.mark.parametrize("shape", [
    LayerShape(2, 512, 256, 5, 7, 256, 128, 3, 1, 1),
    LayerShape(3, 256, 512, 4, 4, 128, 256, 3, 2, 1),
], ids=lambda s: f"{s.C}_{s.N}_{s.H}x{s.W}_s{s.stride}")
def test_3xbf16_split_k_matches_unsplit(env, shape, monkeypatch):
    """Split-K (cluster DSMEM reduction) and the unsplit path agree to rounding, and
    the split result is deterministic run to run (fixed reduction order, R10)."""
    s = shape.with_batch(shape.B)
    d = synth.make_layer(s, seed=5, bias=True)
    monkeypatch.setenv("TDC_SPLITK", "1")
    a, _ = run_layer(env, s, d, "nhwc", "3xbf16")
    b, _ = run_layer(env, s, d, "nhwc", "3xbf16")
    assert np.array_equal(a, b)
    monkeypatch.setenv("TDC_SPLITK", "0")
    c, _ = run_layer(env, s, d, "nhwc", "3xbf16")
    ref = ref_of(s, d)
    assert err(a, ref) <= TOL["3xbf16"] and err(c, ref) <= TOL["3xbf16"]


@pytest.mark.parametrize("shape", [LayerShape(16, 512, 512, 28, 28, 192, 192, 3, 1, 1, "28x28_512_D192_b16")],
                         ids=lambda s: s.name)
def test_3xbf16_wide_rank_large_m(env, shape):
    """Large M with D1 = D2 = 192: the stage-1 N tile must shrink until its rings fit
    shared memory (a Tucker VGG-16 28x28x512 layer at batch 64 hit this).  Sampled
    outputs against the oracle evaluated point by point."""
    d = synth.make_layer(shape, seed=9)
    got, info = run_layer(env, shape, d, "nhwc", "3xbf16")
    assert "3xbf16" in info.variant_name, info.variant_name
    pts = synth.sample_points(shape, 200, seed=1)
    ref = oracle.tkd_points(d["x"], d["core"], d["u_in"], d["u_out"], pts, None, shape.stride, shape.pad)
    vals = np.array([got[p] for p in pts], dtype=np.float64)
    assert np.max(np.abs(vals - ref)) / np.max(np.abs(ref)) <= TOL["3xbf16"]


@pytest.mark.parametrize("gs", [2, 3, 5])
@pytest.mark.parametrize("shape", [
    LayerShape(2, 512, 256, 5, 7, 256, 128, 3, 1, 1),
    LayerShape(3, 256, 512, 4, 4, 128, 256, 3, 2, 1),
    LayerShape(2, 320, 240, 9, 6, 160, 224, 3, 1, 1),
], ids=lambda s: f"{s.C}_{s.N}_{s.H}x{s.W}_s{s.stride}")
def test_3xbf16_l2_split_k(env, shape, gs, monkeypatch):
    """Split-K through L2 (every stage cut into `gs` K pieces, partials reduced by the
    piece-0 CTA in piece order) against the oracle; deterministic run to run; a
    partial batch equals the slice of the full batch bit for bit (the pieces are fixed
    by the plan, not by the batch)."""
    torch, tdc = env
    monkeypatch.setenv("TDC_NO_FUSE3", "1")
    s = shape.with_batch(shape.B)
    d = synth.make_layer(s, seed=17, bias=True)
    hints = dict(gsplit_stage1=gs, gsplit_core=gs, gsplit_stage3=gs)

    def run(batch):
        plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16, hints=hints)
        x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
        y = torch.full((s.B, s.Ho, s.Wo, s.N), float("nan"), device="cuda")
        plan.forward(x, y, batch=batch)
        torch.cuda.synchronize()
        info = plan.info()
        plan.close()
        return synth.nhwc_to_nchw(y.cpu().numpy())[:batch], info

    a, info = run(s.B)
    assert info.gsplit_core > 1 and info.gsplit_stage1 > 1 and info.gsplit_stage3 > 1
    b, _ = run(s.B)
    assert np.array_equal(a, b)
    part, _ = run(1)
    assert np.array_equal(part, a[:1])
    assert err(a, ref_of(s, d)) <= TOL["3xbf16"]


@pytest.mark.parametrize("shape,count", synth.R18_SHAPES[4:], ids=[s.name for s, _ in synth.R18_SHAPES[4:]])
def test_3xbf16_r18_small_layers_planned_split(env, shape, count):
    """The 14x14 / 7x7 ResNet-18 layers at batch 32 (few output tiles, long K) as planned
    (split-K through L2 where the planner picks it), sampled against the oracle."""
    s = shape.with_batch(32)
    d = synth.make_layer(s, seed=2, bias=True)
    got, info = run_layer(env, s, d, "nhwc", "3xbf16")
    pts = synth.sample_points(s, 300, seed=4)
    ref = oracle.tkd_points(d["x"], d["core"], d["u_in"], d["u_out"], pts, d["bias"], s.stride, s.pad)
    vals = np.array([got[p] for p in pts], dtype=np.float64)
    assert np.max(np.abs(vals - ref)) / np.max(np.abs(ref)) <= TOL["3xbf16"]


@pytest.mark.parametrize("math,layout", [("3xbf16", "nhwc"), ("tf32", "nhwc"), ("fp32", "nchw")])
def test_forward_host_pipelined_chunks(env, math, layout):
    """tdc_conv_forward_host splits a large batch into image chunks whose H2D copy,
    forward and D2H copy overlap on three streams; the result equals the device-buffer
    forward of the whole batch bit for bit (images are independent)."""
    torch, tdc = env
    s = synth.R18_SHAPES[0][0].with_batch(8)  # 56x56x64: ~13 MB of traffic -> 6 chunks
    d = synth.make_layer(s, seed=31, bias=True)
    lay = tdc.TDC_LAYOUT_NHWC if layout == "nhwc" else tdc.TDC_LAYOUT_NCHW
    plan = tdc.ConvPlan(s, d, layout=lay, math=tdc.MATH_NAMES[math])
    xn = synth.nchw_to_nhwc(d["x"]) if layout == "nhwc" else np.ascontiguousarray(d["x"])
    yshape = (s.B, s.Ho, s.Wo, s.N) if layout == "nhwc" else (s.B, s.N, s.Ho, s.Wo)
    xh = torch.from_numpy(xn).pin_memory()
    yh = torch.full(yshape, float("nan")).pin_memory()
    plan.forward_host(xh, yh)
    plan.forward_host(xh, yh)  # twice: the pipeline's streams/events are reused
    xd = torch.from_numpy(xn).cuda()
    yd = torch.full(yshape, float("nan"), device="cuda")
    plan.forward(xd, yd)
    torch.cuda.synchronize()
    plan.close()
    assert np.array_equal(yh.numpy(), yd.cpu().numpy())
    ref = ref_of(s, d)
    got = synth.nhwc_to_nchw(yh.numpy()) if layout == "nhwc" else yh.numpy()
    assert err(got, ref) <= TOL[math]


def test_forward_host_many_matches_device(env):
    """tdc_conv_forward_host_many pipelines several layers' host-buffer forwards in one
    call; each result equals that layer's device-buffer forward bit for bit."""
    torch, tdc = env
    shapes = [synth.R18_SHAPES[i][0].with_batch(b) for i, b in ((0, 4), (4, 8), (6, 3), (1, 2))]
    plans, xs, ys, refs = [], [], [], []
    for k, s in enumerate(shapes):
        d = synth.make_layer(s, seed=40 + k, bias=True)
        p = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16)
        xn = synth.nchw_to_nhwc(d["x"])
        xd = torch.from_numpy(xn).cuda()
        yd = torch.full((s.B, s.Ho, s.Wo, s.N), float("nan"), device="cuda")
        p.forward(xd, yd)
        refs.append(yd)
        plans.append(p)
        xs.append(torch.from_numpy(xn).pin_memory())
        ys.append(torch.full((s.B, s.Ho, s.Wo, s.N), float("nan")).pin_memory())
    tdc.forward_host_many(plans, xs, ys)
    tdc.forward_host_many(plans, xs, ys)
    torch.cuda.synchronize()
    for y, r in zip(ys, refs):
        assert np.array_equal(y.numpy(), r.cpu().numpy())
    for p in plans:
        p.close()


# Batch 1 (the paper's regime, P:L509 / P:L595): the 56x56 layer runs the TMEM-operand
# single-launch kernel, every other R18 shape a latency-mode three-launch plan (32-wide N
# tiles, core K split over a 4-CTA cluster).  Full outputs against the oracle.
@pytest.mark.parametrize("idx", range(len(synth.R18_SHAPES)))
@pytest.mark.parametrize("bias", [False, True])
def test_batch1_plans_match_oracle(env, idx, bias):
    shape = synth.R18_SHAPES[idx][0].with_batch(1)
    d = synth.make_layer(shape, layer_id=40 + idx, bias=bias)
    got, info = run_layer(env, shape, d, math="3xbf16")
    if idx == 0:
        assert info.variant_name == "layer_3xbf16_fused"
    else:
        assert info.variant_name == "tc3_3xbf16_band", info.variant_name
        assert info.bn_core == 32 and info.bn_stage1 == 32 and info.bn_stage3 == 32
        assert info.ksplit_core == min(4, (shape.D1 + 31) // 32)  # the cluster splits whole 32-channel chunks
    e = err(got, ref_of(shape, d))
    assert e <= TOL["3xbf16"], (shape.name, info.variant_name, e)


def test_batch32_plans_are_not_latency_mode(env):
    # the bench-batch plans keep the throughput tiling (no forced cluster split of the core)
    torch, tdc = env
    for shape, _ in synth.R18_SHAPES[1:]:
        s = shape.with_batch(32)
        plan = tdc.ConvPlan(s, synth.make_layer(s), math=tdc.TDC_MATH_3XBF16)
        info = plan.info()
        plan.close()
        assert info.ksplit_core == 1, (s.name, info)


# Stage 2 on CTA pairs (cta_group::2, tdc_bf_core2_kernel): streamed-weight 3x3 cores.
# Odd M-tile counts (a phantom tile in the last pair), ragged ranks, a smaller
# batch than planned, bias; against the oracle and run to run bit-identical.
@pytest.mark.parametrize("shape", [
    LayerShape(9, 256, 256, 10, 10, 256, 256, 3, 1, 1),   # 11 M tiles: phantom tile in the last pair
    LayerShape(10, 192, 320, 9, 11, 160, 224, 3, 1, 1),   # ragged ranks / channels
    synth.R18_SHAPES[6][0].with_batch(32),                 # the 7x7 R18 layer at the bench batch
], ids=lambda s: f"{s.B}x{s.C}x{s.H}x{s.W}_D{s.D1}-{s.D2}_s{s.stride}")
def test_core_on_cta_pairs(env, shape):
    torch, tdc = env
    d = synth.make_layer(shape, seed=33, bias=True)
    plan = tdc.ConvPlan(shape, d, math=tdc.TDC_MATH_3XBF16)
    info = plan.info()
    plan.close()
    if info.variant_name != "tc3_3xbf16_pair":
        pytest.skip(f"planner chose {info.variant_name} for this shape")
    for b in sorted({shape.B, max(1, shape.B - 1), 1}, reverse=True):  # batch 1: one M tile, a phantom peer
        got, info = run_layer(env, shape, d, math="3xbf16", batch=b)
        assert info.variant_name == "tc3_3xbf16_pair"
        e = err(got, ref_of(shape, d, b))
        assert e <= TOL["3xbf16"], (shape, b, e)
        again, _ = run_layer(env, shape, d, math="3xbf16", batch=b)
        assert np.array_equal(got, again)


# The paper's two weak VGG-16 shapes as TKD layers at batch 1: full outputs
# against the oracle in the headline math mode.
@pytest.mark.parametrize("shape", synth.PAPER_WEAK_SHAPES, ids=lambda s: s.name)
def test_paper_weak_vgg_shapes(env, shape):
    d = synth.make_layer(shape, layer_id=60, bias=True)
    got, info = run_layer(env, shape, d, math="3xbf16")
    e = err(got, ref_of(shape, d))
    assert e <= TOL["3xbf16"], (shape.name, info.variant_name, e)


def test_wide_rank_stage1_large_batch(env):
    # Tucker VGG-16 conv4 (28x28, C = N = 512, D = 192) at batch 64: the stage-1 N tile is
    # capped at 128 (two accumulators + two TMEM X slots in 512 columns); images 0 and 63
    # against the oracle
    torch, tdc = env
    s = LayerShape(64, 512, 512, 28, 28, 192, 192, 3, 1, 1, "vgg_28_512_r192_b64")
    d = synth.make_layer(s, seed=71, bias=True)
    plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16)
    assert plan.info().bn_stage1 <= 128
    x = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
    y = torch.empty((s.B, s.Ho, s.Wo, s.N), device="cuda")
    plan.forward(x, y)
    torch.cuda.synchronize()
    got = synth.nhwc_to_nchw(y.cpu().numpy())
    plan.close()
    for i in (0, 63):
        ref = oracle.tkd_stages(d["x"][i:i + 1], d["core"], d["u_in"], d["u_out"], d["bias"], s.stride, s.pad)
        assert err(got[i:i + 1], ref) <= TOL["3xbf16"], i
