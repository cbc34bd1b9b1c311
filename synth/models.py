"""Seeded synthetic Tucker ResNet-18 / ResNet-50 / VGG-16 op lists (SURVEY §8(d)
configs 3-4, §8(f) NEXT-1) in the model C-ABI's op vocabulary (include/tdc.h).

Like ``synth/__init__``, this module only lays out architectures and draws random
weights; it contains none of the method's arithmetic.  Every 3x3 convolution except
the stem is a TKD layer with "paper-style" ranks D = ceil(r * C), D2 = ceil(r * N)
(reading A15: r = 1/2 for ResNet-18, 1/4 for ResNet-50, 3/8 for VGG-16); the stem,
1x1 convolutions and the classifier stay dense ("use cuDNN to implement other
layers").  Each conv is followed by BN (random gamma, beta, running mean/var) that the
runtime folds; ReLU and the residual add are op flags.

Weights: dense conv He-normal N(0, 2 / (C K^2)); TKD factors as ``synth.make_layer``
(orthonormal U, core N(0, 2 / (D1 K^2))); BN gamma ~ U[0.8, 1.2), beta ~ U[-0.1, 0.1),
mean ~ U[-0.1, 0.1), var ~ U[0.8, 1.2); FC N(0, 1 / C) and bias U[-0.1, 0.1).
Seeds: PCG64(seed + 1000 * op index + tensor offset).
"""
from __future__ import annotations

import math

import numpy as np

from . import _orthonormal

OP_CONV, OP_TKD, OP_MAXPOOL, OP_AVGPOOL, OP_FC = 0, 1, 2, 3, 4


def _rng(seed, i, off):
    return np.random.Generator(np.random.PCG64(seed + 1000 * i + off))


class _Builder:
    def __init__(self, seed, H, W, C):
        self.seed, self.ops = seed, []
        self.geo = {0: (H, W, C)}  # id -> (H, W, C)

    def _add(self, op, Ho, Wo, Co):
        self.ops.append(op)
        nid = len(self.ops)
        self.geo[nid] = (Ho, Wo, Co)
        return nid

    def _bn(self, i, n):
        r = _rng(self.seed, i, 7)
        return np.stack([r.uniform(0.8, 1.2, n), r.uniform(-0.1, 0.1, n), r.uniform(-0.1, 0.1, n),
                         r.uniform(0.8, 1.2, n)]).astype(np.float32)

    def conv(self, src, cout, k, s, p, relu=True, res=-1, tkd_ratio=None, tkd_ranks=None):
        H, W, C = self.geo[src]
        i = len(self.ops)
        Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
        op = {"kind": OP_CONV, "src": src, "res": res, "c_in": C, "c_out": cout, "height": H, "width": W,
              "kernel": k, "stride": s, "pad": p, "rank_in": 0, "rank_out": 0, "relu": int(relu),
              "bias": None, "bn": self._bn(i, cout)}
        if tkd_ratio is not None or tkd_ranks is not None:
            if tkd_ranks is not None:  # per-layer (D1, D2), e.g. from hardware-aware rank selection
                d1, d2 = int(tkd_ranks[0]), int(tkd_ranks[1])
            else:
                d1, d2 = max(1, math.ceil(tkd_ratio * C)), max(1, math.ceil(tkd_ratio * cout))
            op.update(kind=OP_TKD, rank_in=d1, rank_out=d2)
            op["u_in"] = _orthonormal(_rng(self.seed, i, 1), C, d1).astype(np.float32)
            op["w"] = (_rng(self.seed, i, 2).standard_normal((d2, d1, k, k)) *
                       np.sqrt(2.0 / (d1 * k * k))).astype(np.float32)
            op["u_out"] = _orthonormal(_rng(self.seed, i, 3), cout, d2).astype(np.float32)
        else:
            op["w"] = (_rng(self.seed, i, 2).standard_normal((cout, C, k, k)) *
                       np.sqrt(2.0 / (C * k * k))).astype(np.float32)
        return self._add(op, Ho, Wo, cout)

    def maxpool(self, src, k, s, p):
        H, W, C = self.geo[src]
        Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
        return self._add({"kind": OP_MAXPOOL, "src": src, "res": -1, "c_in": C, "c_out": C, "height": H,
                          "width": W, "kernel": k, "stride": s, "pad": p, "relu": 0}, Ho, Wo, C)

    def avgpool(self, src):
        H, W, C = self.geo[src]
        return self._add({"kind": OP_AVGPOOL, "src": src, "res": -1, "c_in": C, "c_out": C, "height": H,
                          "width": W, "kernel": 1, "stride": 1, "pad": 0, "relu": 0}, 1, 1, C)

    def fc(self, src, n):
        _, _, C = self.geo[src]
        i = len(self.ops)
        w = (_rng(self.seed, i, 2).standard_normal((n, C)) / np.sqrt(C)).astype(np.float32)
        b = _rng(self.seed, i, 4).uniform(-0.1, 0.1, n).astype(np.float32)
        return self._add({"kind": OP_FC, "src": src, "res": -1, "c_in": C, "c_out": n, "height": 1, "width": 1,
                          "kernel": 1, "stride": 1, "pad": 0, "relu": 0, "w": w, "bias": b, "bn": None}, 1, 1, n)


def tkd_layer_name(depth: int, H: int, C: int, N: int, s: int) -> str:
    """Shape key of a TKD layer, the names of ranksel.resnet18_layers() (r18_56_64_64_s1 ...)."""
    return f"r{depth}_{H}_{C}_{N}_s{s}"


def tucker_resnet(depth: int = 18, image: int = 224, num_classes: int = 1000, ratio: float | None = None,
                  seed: int = 42, width: int = 64, ranks: dict | None = None):
    """Op list of a Tucker ResNet-18 (basic blocks) or -50 (bottlenecks).  `width` scales
    every stage (64 = the real network; tests use smaller widths).  `ranks` maps a TKD
    layer's shape key (tkd_layer_name, or "<C>_<N>_s<s>" for any image size) to its
    (D1, D2) -- the per-layer plan of hardware-aware rank selection; layers
    it does not name use the uniform ratio."""
    if depth not in (18, 50):
        raise ValueError("depth must be 18 or 50")
    r = ratio if ratio is not None else (0.5 if depth == 18 else 0.25)
    b = _Builder(seed, image, image, 3)

    def rk(src, cin, cout, s):
        if not ranks:
            return None
        H = b.geo[src][0]
        return ranks.get(tkd_layer_name(depth, H, cin, cout, s)) or ranks.get(f"{cin}_{cout}_s{s}")
    x = b.conv(0, width, 7, 2, 3)                       # stem (dense), BN, ReLU
    x = b.maxpool(x, 3, 2, 1)
    blocks = [2, 2, 2, 2] if depth == 18 else [3, 4, 6, 3]
    expansion = 1 if depth == 18 else 4
    cin = width
    for stage, nb in enumerate(blocks):
        planes = width * (2 ** stage)
        for j in range(nb):
            s = 2 if (stage > 0 and j == 0) else 1
            cout = planes * expansion
            shortcut = x
            if s != 1 or cin != cout:
                shortcut = b.conv(x, cout, 1, s, 0, relu=False)          # downsample 1x1 (dense) + BN
            if depth == 18:
                y = b.conv(x, planes, 3, s, 1, tkd_ratio=r, tkd_ranks=rk(x, cin, planes, s))  # TKD + BN + ReLU
                x = b.conv(y, cout, 3, 1, 1, relu=True, res=shortcut, tkd_ratio=r,
                           tkd_ranks=rk(y, planes, cout, 1))                                # + add + ReLU
            else:
                y = b.conv(x, planes, 1, 1, 0)                           # 1x1 (dense) + BN + ReLU
                y = b.conv(y, planes, 3, s, 1, tkd_ratio=r, tkd_ranks=rk(y, planes, planes, s))  # TKD + BN + ReLU
                x = b.conv(y, cout, 1, 1, 0, relu=True, res=shortcut)    # 1x1 (dense) + BN + add + ReLU
            cin = cout
    x = b.avgpool(x)
    b.fc(x, num_classes)
    return b.ops


def tucker_vgg16(image: int = 224, num_classes: int = 1000, ratio: float = 3 / 8, seed: int = 42,
                 width: int = 64, hidden: int = 4096):
    """Op list of a Tucker VGG-16 (BN variant): the first 3x3 conv dense, the other 12
    TKD with r = 3/8 (reading A15); classifier = a dense (image/32) x (image/32) conv
    (FC1 on the flattened NHWC feature map), FC2, FC3."""
    b = _Builder(seed, image, image, 3)
    cfg = [1, 1, "M", 2, 2, "M", 4, 4, 4, "M", 8, 8, 8, "M", 8, 8, 8, "M"]
    x, first = 0, True
    for v in cfg:
        if v == "M":
            x = b.maxpool(x, 2, 2, 0)
            continue
        x = b.conv(x, width * v, 3, 1, 1, tkd_ratio=None if first else ratio)
        first = False
    h, _, _ = b.geo[x]
    x = b.conv(x, hidden, h, 1, 0)                       # FC1 as a valid conv over the feature map
    b.ops[-1]["bn"] = None
    b.ops[-1]["bias"] = _rng(seed, len(b.ops) - 1, 4).uniform(-0.1, 0.1, hidden).astype(np.float32)
    x = b.fc(x, hidden)
    b.ops[-1]["relu"] = 1
    b.fc(x, num_classes)
    return b.ops


def model_input(batch: int, image: int = 224, seed: int = 42, first: int = 0) -> np.ndarray:
    """Synthetic ImageNet-shaped input, NHWC fp32 ~ N(0, 1) (normalised pixels):
    images [first, first + batch) of the global batch, one seeded stream per image so
    a rank's shard equals the same slice of the unsharded batch."""
    out = np.empty((batch, image, image, 3), np.float32)
    for i in range(batch):
        g = np.random.Generator(np.random.PCG64([seed, 999_999, first + i]))
        out[i] = g.standard_normal((image, image, 3)).astype(np.float32)
    return out
