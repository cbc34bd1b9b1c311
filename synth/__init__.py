"""Seeded synthetic inputs for the TKD layer (shared by tests, bench and smoke).

This module holds workload definitions and random-number recipes only; it
contains none of the method's arithmetic (no convolution, no contraction).
Both the fp64 oracle and the CUDA path receive exactly the fp32 arrays made
here.  Recipe:

* numpy ``Generator(PCG64(seed))``, base seed 42, per-tensor offset
  x=0, u_in=1, core=2, u_out=3, bias=4, plus 16 x layer id;
* x ~ U[-1, 1); U_in, U_out = first D columns of Q from a QR of a Gaussian
  (orthonormal, as truncated HOSVD produces); core ~ N(0, 2/(D1 K^2));
* ``integer=True``: every tensor uniform on {-2..2}; all partial sums are then
  integers far below 2^24, exact in fp32 (SURVEY §8(c) pin 8).
"""
from __future__ import annotations

from dataclasses import dataclass, asdict

import numpy as np

BASE_SEED = 42


@dataclass(frozen=True)
class LayerShape:
    """One TKD layer: input B x C x H x W, core D2 x D1 x K x K, output N channels."""
    B: int
    C: int
    N: int
    H: int
    W: int
    D1: int
    D2: int
    K: int = 3
    stride: int = 1
    pad: int = 1
    name: str = ""

    @property
    def Ho(self) -> int:
        return (self.H + 2 * self.pad - self.K) // self.stride + 1

    @property
    def Wo(self) -> int:
        return (self.W + 2 * self.pad - self.K) // self.stride + 1

    def with_batch(self, B: int) -> "LayerShape":
        d = asdict(self)
        d["B"] = B
        return LayerShape(**d)

    def as_dict(self) -> dict:
        return asdict(self)


# BASELINE.json configs[0]: batch 1, C=N=16, D1=D2=4, 3x3 core, 8x8, s=1, p=1.
CONFIG1 = LayerShape(B=1, C=16, N=16, H=8, W=8, D1=4, D2=4, K=3, stride=1, pad=1,
                     name="config1")

# BASELINE.json configs[1]: the 3x3 conv shapes of ResNet-18 with paper-style
# ranks D1 = C/2, D2 = N/2 (reading R15).  (shape, count in R18)
R18_SHAPES = [
    (LayerShape(1, 64, 64, 56, 56, 32, 32, 3, 1, 1, "r18_56_64_64_s1"), 4),
    (LayerShape(1, 64, 128, 56, 56, 32, 64, 3, 2, 1, "r18_56_64_128_s2"), 1),
    (LayerShape(1, 128, 128, 28, 28, 64, 64, 3, 1, 1, "r18_28_128_128_s1"), 3),
    (LayerShape(1, 128, 256, 28, 28, 64, 128, 3, 2, 1, "r18_28_128_256_s2"), 1),
    (LayerShape(1, 256, 256, 14, 14, 128, 128, 3, 1, 1, "r18_14_256_256_s1"), 3),
    (LayerShape(1, 256, 512, 14, 14, 128, 256, 3, 2, 1, "r18_14_256_512_s2"), 1),
    (LayerShape(1, 512, 512, 7, 7, 256, 256, 3, 1, 1, "r18_7_512_512_s1"), 3),
]

# The two VGG-16 core-convolution shapes the paper names as its weak cases (P:L599-602:
# "(64, 32, 224, 224) and (64, 32, 112, 112) ... slower than or similar to TVM and cuDNN"),
# read as core D1 = 64 -> D2 = 32 at H = W = 224 / 112 inside the VGG-16 block's C = N = 64 /
# 128 layer, batch 1 (the paper's kernel-evaluation batch).
PAPER_WEAK_SHAPES = [
    LayerShape(1, 64, 64, 224, 224, 64, 32, 3, 1, 1, "vgg_224_64_64_core64x32"),
    LayerShape(1, 128, 128, 112, 112, 64, 32, 3, 1, 1, "vgg_112_128_128_core64x32"),
]

# BASELINE.json configs[4]: rank sweep on a 28x28x256 -> 256 3x3 layer.
RANK_GRID = (8, 16, 32, 64, 128)


def rank_sweep_shape(D1: int, D2: int, B: int = 1) -> LayerShape:
    return LayerShape(B, 256, 256, 28, 28, D1, D2, 3, 1, 1, f"sweep_{D1}_{D2}")


def _rng(seed: int, layer_id: int, offset: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed + 16 * layer_id + offset))


def _orthonormal(rng: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    g = rng.standard_normal((rows, max(cols, 1)))
    q, r = np.linalg.qr(g)
    # sign fix for determinism across LAPACK builds: diag(R) >= 0
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return (q * s)[:, :cols]


def make_layer(shape: LayerShape, seed: int = BASE_SEED, layer_id: int = 0,
               integer: bool = False, bias: bool = False) -> dict:
    """fp32 arrays: x (B,C,H,W NCHW), core (D2,D1,K,K), u_in (C,D1), u_out (N,D2), bias (N)|None."""
    s = shape
    if integer:
        ints = lambda off, shp: _rng(seed, layer_id, off).integers(-2, 3, size=shp).astype(np.float32)
        x = ints(0, (s.B, s.C, s.H, s.W))
        u_in = ints(1, (s.C, s.D1))
        core = ints(2, (s.D2, s.D1, s.K, s.K))
        u_out = ints(3, (s.N, s.D2))
        b = ints(4, (s.N,)) if bias else None
    else:
        x = _rng(seed, layer_id, 0).uniform(-1.0, 1.0, (s.B, s.C, s.H, s.W)).astype(np.float32)
        u_in = _orthonormal(_rng(seed, layer_id, 1), s.C, s.D1).astype(np.float32) \
            if s.D1 <= s.C else _rng(seed, layer_id, 1).standard_normal((s.C, s.D1)).astype(np.float32)
        core = (_rng(seed, layer_id, 2).standard_normal((s.D2, s.D1, s.K, s.K))
                * np.sqrt(2.0 / (s.D1 * s.K * s.K))).astype(np.float32)
        u_out = _orthonormal(_rng(seed, layer_id, 3), s.N, s.D2).astype(np.float32) \
            if s.D2 <= s.N else _rng(seed, layer_id, 3).standard_normal((s.N, s.D2)).astype(np.float32)
        b = _rng(seed, layer_id, 4).uniform(-0.1, 0.1, (s.N,)).astype(np.float32) if bias else None
    return {"x": np.ascontiguousarray(x), "core": np.ascontiguousarray(core),
            "u_in": np.ascontiguousarray(u_in), "u_out": np.ascontiguousarray(u_out),
            "bias": b}


def make_images(shape: LayerShape, first: int, count: int, seed: int = BASE_SEED,
                layer_id: int = 0) -> np.ndarray:
    """Images [first, first + count) of a layer's global input batch, NCHW fp32
    ~ U[-1, 1): every image has its own counter-based stream (seed, layer, image), so a
    rank's shard of the global batch is the same data whatever the number of ranks
    (multi-GPU runs shard the batch)."""
    s = shape
    out = np.empty((count, s.C, s.H, s.W), np.float32)
    for i in range(count):
        g = np.random.Generator(np.random.PCG64([seed, layer_id, 0x1A6E, first + i]))
        out[i] = g.uniform(-1.0, 1.0, (s.C, s.H, s.W)).astype(np.float32)
    return out


def nchw_to_nhwc(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.transpose(a, (0, 2, 3, 1)))


def nhwc_to_nchw(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.transpose(a, (0, 3, 1, 2)))


def sample_points(shape: LayerShape, count: int, seed: int = BASE_SEED) -> list:
    """Seeded (b, n, i, j) output coordinates, always including the four corners
    of the first and last image (padding-boundary cases) and the ragged tail."""
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    pts = set()
    for b in {0, shape.B - 1}:
        for i in {0, shape.Ho - 1}:
            for j in {0, shape.Wo - 1}:
                pts.add((b, int(rng.integers(shape.N)), i, j))
    pts.add((shape.B - 1, shape.N - 1, shape.Ho - 1, shape.Wo - 1))
    while len(pts) < count:
        pts.add((int(rng.integers(shape.B)), int(rng.integers(shape.N)),
                 int(rng.integers(shape.Ho)), int(rng.integers(shape.Wo))))
    return sorted(pts)
