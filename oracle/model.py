"""fp64 oracle of the whole-model path (TEST INFRASTRUCTURE ONLY -- like the rest of
oracle/, only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline may use it).

Follows the op semantics of include/tdc.h "models" literally, op by op, with nothing
folded: conv / TKD / FC, then + bias, then BatchNorm with its running statistics
(y - mean) / sqrt(var + 1e-5) * gamma + beta, then + residual, then ReLU.  Convolutions
use the seven-loop oracle (``oracle.conv7``, cross-correlation, reading R4) and TKD
layers the three-stage oracle (``oracle.tkd_stages``).  Activations are NCHW fp64.
"""
from __future__ import annotations

import numpy as np

from . import conv7, tkd_stages

OP_CONV, OP_TKD, OP_MAXPOOL, OP_AVGPOOL, OP_FC = 0, 1, 2, 3, 4
BN_EPS = 1e-5


def maxpool(x: np.ndarray, k: int, s: int, p: int) -> np.ndarray:
    B, C, H, W = x.shape
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    xp = np.full((B, C, H + 2 * p, W + 2 * p), -np.inf)
    xp[:, :, p:p + H, p:p + W] = x
    y = np.full((B, C, Ho, Wo), -np.inf)
    for r in range(k):
        for t in range(k):
            y = np.maximum(y, xp[:, :, r:r + s * (Ho - 1) + 1:s, t:t + s * (Wo - 1) + 1:s])
    return y


def forward(ops: list, x_nhwc: np.ndarray) -> np.ndarray:
    """Model output for input x (B x H x W x C, NHWC); returns NHWC fp64."""
    acts = {0: np.ascontiguousarray(np.transpose(np.asarray(x_nhwc, np.float64), (0, 3, 1, 2)))}
    for i, o in enumerate(ops):
        x = acts[o["src"]]
        k = o["kind"]
        if k == OP_CONV:
            y = conv7(x, o["w"], o["stride"], o["pad"])
        elif k == OP_TKD:
            y = tkd_stages(x, o["w"], o["u_in"], o["u_out"], None, o["stride"], o["pad"])
        elif k == OP_MAXPOOL:
            y = maxpool(x, o["kernel"], o["stride"], o["pad"])
        elif k == OP_AVGPOOL:
            y = x.mean(axis=(2, 3), keepdims=True)
        elif k == OP_FC:
            y = (x.reshape(x.shape[0], -1) @ np.asarray(o["w"], np.float64).T)[:, :, None, None]
        else:
            raise ValueError(f"op {i}: unknown kind {k}")
        if k in (OP_CONV, OP_TKD, OP_FC):
            if o.get("bias") is not None:
                y = y + np.asarray(o["bias"], np.float64)[None, :, None, None]
            if o.get("bn") is not None:
                g, b, m, v = (np.asarray(a, np.float64)[None, :, None, None] for a in o["bn"])
                y = (y - m) / np.sqrt(v + BN_EPS) * g + b
            if o.get("res", -1) >= 0:
                y = y + acts[o["res"]]
            if o.get("relu"):
                y = np.maximum(y, 0.0)
        acts[i + 1] = y
    return np.ascontiguousarray(np.transpose(acts[len(ops)], (0, 2, 3, 1)))
