"""Whole-model path: the fp64 model oracle pinned against torch
fp64 reference ops, and (GPU) Tucker ResNet-18/-50 through tdc_model_forward against it.

Model tolerance (reading R19): max-normalized error <= 1e-3 on the model
output -- every TKD / dense layer is fp32-grade (3xBF16, <= 1e-4 each) and the error
compounds over up to 54 layers."""
import numpy as np
import pytest

import oracle
import oracle.model as om
import synth
import synth.models as sm

MODEL_TOL = 1e-3


def torch_ref(ops, x_nhwc):
    """Independent fp64 reference of the op list with torch.nn.functional."""
    import torch
    import torch.nn.functional as F
    acts = {0: torch.from_numpy(np.transpose(x_nhwc, (0, 3, 1, 2)).astype(np.float64))}
    for i, o in enumerate(ops):
        x = acts[o["src"]]
        k = o["kind"]
        if k == sm.OP_CONV:
            y = F.conv2d(x, torch.from_numpy(o["w"].astype(np.float64)), stride=o["stride"], padding=o["pad"])
        elif k == sm.OP_TKD:
            w = np.einsum("nq,qart,ca->ncrt", o["u_out"].astype(np.float64), o["w"].astype(np.float64),
                          o["u_in"].astype(np.float64))
            y = F.conv2d(x, torch.from_numpy(w), stride=o["stride"], padding=o["pad"])
        elif k == sm.OP_MAXPOOL:
            y = F.max_pool2d(x, o["kernel"], o["stride"], o["pad"])
        elif k == sm.OP_AVGPOOL:
            y = F.adaptive_avg_pool2d(x, 1)
        else:
            y = F.linear(x.flatten(1), torch.from_numpy(o["w"].astype(np.float64)))[:, :, None, None]
        if k in (sm.OP_CONV, sm.OP_TKD, sm.OP_FC):
            if o.get("bias") is not None:
                y = y + torch.from_numpy(o["bias"].astype(np.float64))[None, :, None, None]
            if o.get("bn") is not None:
                g, b, m, v = (torch.from_numpy(a.astype(np.float64)) for a in o["bn"])
                y = F.batch_norm(y, m, v, g, b, training=False, eps=1e-5)
            if o.get("res", -1) >= 0:
                y = y + acts[o["res"]]
            if o.get("relu"):
                y = torch.relu(y)
        acts[i + 1] = y
    return np.transpose(acts[len(ops)].numpy(), (0, 2, 3, 1))


def maxerr(got, ref):
    return float(np.max(np.abs(np.asarray(got, np.float64) - ref)) / np.max(np.abs(ref)))


@pytest.mark.parametrize("arch", ["r18", "r50", "vgg16"])
def test_model_oracle_against_torch(arch):
    ops = (sm.tucker_vgg16(image=32, num_classes=10, width=8, hidden=64) if arch == "vgg16"
           else sm.tucker_resnet(18 if arch == "r18" else 50, image=32, num_classes=10, width=8))
    x = sm.model_input(2, 32)
    assert maxerr(om.forward(ops, x), torch_ref(ops, x)) < 1e-12


def test_model_oracle_pool_semantics():
    x = np.arange(2 * 5 * 5 * 3, dtype=np.float64).reshape(2, 3, 5, 5) - 40
    y = om.maxpool(x, 3, 2, 1)
    assert y.shape == (2, 3, 3, 3)
    assert y[0, 0, 0, 0] == max(x[0, 0, 0, 0], x[0, 0, 0, 1], x[0, 0, 1, 0], x[0, 0, 1, 1])  # padding never wins
    assert y[1, 2, 2, 2] == x[1, 2, 4, 4]


def test_builder_geometry_and_ranks():
    ops = sm.tucker_resnet(18)
    tkd = [o for o in ops if o["kind"] == sm.OP_TKD]
    assert len(tkd) == 16 and all(o["rank_in"] == o["c_in"] // 2 for o in tkd)   # paper-style r = 1/2
    ops50 = sm.tucker_resnet(50)
    assert sum(o["kind"] == sm.OP_TKD for o in ops50) == 16
    vgg = sm.tucker_vgg16()
    assert sum(o["kind"] == sm.OP_TKD for o in vgg) == 12
    assert all(o["rank_in"] == -(-3 * o["c_in"] // 8) for o in vgg if o["kind"] == sm.OP_TKD)
    assert sum(o["kind"] == sm.OP_CONV and o["kernel"] == 1 for o in ops50) == 36  # 32 + 4 downsample
    assert ops50[-1]["kind"] == sm.OP_FC and ops50[-1]["c_out"] == 1000


def test_builder_per_layer_ranks():
    """Per-layer ranks of a rank plan (NEXT-2) reach the op list: shape keys at the real
    image size, "<C>_<N>_s<s>" keys at any size, the uniform ratio elsewhere."""
    plan = {"r18_56_64_64_s1": (16, 24), "r18_7_512_512_s1": (128, 192)}
    ops = sm.tucker_resnet(18, ranks=plan)
    tkd = [o for o in ops if o["kind"] == sm.OP_TKD]
    got = {(o["height"], o["c_in"], o["c_out"], o["stride"]): (o["rank_in"], o["rank_out"]) for o in tkd}
    assert got[(56, 64, 64, 1)] == (16, 24) and got[(7, 512, 512, 1)] == (128, 192)
    assert got[(28, 128, 128, 1)] == (64, 64)                       # not in the plan: r = 1/2
    for o in tkd:
        assert o["u_in"].shape == (o["c_in"], o["rank_in"]) and o["u_out"].shape == (o["c_out"], o["rank_out"])
        assert o["w"].shape == (o["rank_out"], o["rank_in"], 3, 3)
    small = sm.tucker_resnet(18, image=32, width=8, ranks={"8_8_s1": (3, 5)})
    assert all((o["rank_in"], o["rank_out"]) == (3, 5) for o in small
               if o["kind"] == sm.OP_TKD and o["c_in"] == 8 and o["c_out"] == 8 and o["stride"] == 1)


def latest_rank_plan():
    import glob
    import json
    import os
    paths = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "..", "profiles", "r*_rank_plan_r18_b32.json")))
    if not paths:
        return None
    with open(paths[-1]) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2211_03715_b200 import tdc
    return torch, tdc


def run_model(gpu, ops, x, batch=None):
    torch, tdc = gpu
    m = tdc.Model(ops, max_batch=x.shape[0])
    h, w, c = m.output_shape()
    b = x.shape[0] if batch is None else batch
    xd = torch.from_numpy(x).cuda()
    out = torch.full((x.shape[0], h, w, c), float("nan"), device="cuda")
    m.forward(xd, out, batch=b)
    torch.cuda.synchronize()
    m.close()
    return out.cpu().numpy()[:b]


@pytest.mark.gpu
@pytest.mark.parametrize("depth,width,image", [(18, 16, 32), (50, 16, 32), (18, 32, 64)])
def test_small_tucker_resnet(gpu, depth, width, image):
    ops = sm.tucker_resnet(depth, image=image, num_classes=37, width=width, seed=7)
    x = sm.model_input(3, image, seed=7)
    assert maxerr(run_model(gpu, ops, x), om.forward(ops, x)) <= MODEL_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["greedy", "exact"])
def test_tucker_resnet18_with_selected_ranks(gpu, method):
    """NEXT-2 closed: a Tucker ResNet-18 built with the ranks the hardware-aware selection
    picked from the measured B200 tables (profiles/r*_rank_plan_r18_b32.json), full size,
    through tdc_model_forward, against the fp64 model oracle."""
    plan = latest_rank_plan()
    if plan is None:
        pytest.skip("no rank plan in profiles/")
    ranks = {k: tuple(v) for k, v in plan[method]["ranks"].items()}
    ops = sm.tucker_resnet(18, ranks=ranks)
    tkd = [o for o in ops if o["kind"] == sm.OP_TKD]
    assert any((o["rank_in"], o["rank_out"]) != (o["c_in"] // 2, o["c_out"] // 2) for o in tkd) or \
        all(tuple(v) == (int(k.split("_")[2]) // 2, int(k.split("_")[3]) // 2) for k, v in ranks.items())
    x = sm.model_input(2, 224, seed=11)
    got = run_model(gpu, ops, x)
    assert maxerr(got, om.forward(ops, x)) <= MODEL_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("depth", [18, 50])
def test_full_tucker_resnet_224(gpu, depth):
    """BASELINE config 3 architecture at full size (224 x 224 x 3, 1000 classes)."""
    ops = sm.tucker_resnet(depth)
    x = sm.model_input(2, 224)
    got = run_model(gpu, ops, x)
    assert got.shape == (2, 1, 1, 1000)
    assert maxerr(got, om.forward(ops, x)) <= MODEL_TOL


@pytest.mark.gpu
def test_small_tucker_vgg16(gpu):
    ops = sm.tucker_vgg16(image=64, num_classes=21, width=16, hidden=128, seed=3)
    x = sm.model_input(3, 64, seed=3)
    assert maxerr(run_model(gpu, ops, x), om.forward(ops, x)) <= MODEL_TOL


@pytest.mark.gpu
def test_full_tucker_vgg16_224(gpu):
    """BASELINE config 4 architecture at full size (one image per shard)."""
    ops = sm.tucker_vgg16()
    x = sm.model_input(1, 224, seed=5)
    assert maxerr(run_model(gpu, ops, x), om.forward(ops, x)) <= MODEL_TOL


@pytest.mark.gpu
def test_model_partial_batch_and_determinism(gpu):
    ops = sm.tucker_resnet(18, image=32, num_classes=10, width=16)
    x = sm.model_input(4, 32)
    full = run_model(gpu, ops, x)
    part = run_model(gpu, ops, x, batch=2)
    assert np.array_equal(full[:2], part)
    assert np.array_equal(full, run_model(gpu, ops, x))


@pytest.mark.gpu
def test_model_rejects_bad_graphs(gpu):
    torch, tdc = gpu
    ops = sm.tucker_resnet(18, image=32, num_classes=10, width=16)
    bad = [dict(o) for o in ops]
    bad[3]["src"] = 7            # refers to a later op
    with pytest.raises(tdc.TdcError):
        tdc.Model(bad, 2)
    bad = [dict(o) for o in ops]
    bad[2]["c_in"] += 4          # geometry mismatch with its source
    with pytest.raises(tdc.TdcError):
        tdc.Model(bad, 2)


@pytest.mark.gpu
def test_vgg16_classifier_split_k_partial_batch_and_determinism(gpu):
    """The VGG-16 classifier GEMMs (one M tile, K up to 25,088) run split-K through L2
    (fixed pieces per plan): a partial batch equals the slice of the full batch bit for
    bit and repeated forwards are identical."""
    ops = sm.tucker_vgg16()
    x = sm.model_input(3, 224, seed=11)
    full = run_model(gpu, ops, x)
    assert np.array_equal(full[:2], run_model(gpu, ops, x, batch=2))
    assert np.array_equal(full, run_model(gpu, ops, x))
