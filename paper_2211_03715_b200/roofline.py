"""Algorithmic work of a TKD layer and the B200 roofline denominators.

Host-side accounting used by bench.py and the tests (no device work).

Per layer forward:
  FLOPs = 2 B (H W C D1 + H' W' D1 D2 K^2 + H' W' D2 N)          (1 MAC = 2 FLOPs)
  bytes = 4 B (H W C + H' W' N) + 4 (C D1 + D1 D2 K^2 + D2 N [+ N])  (fused: x in, y out,
                                                                   weights once)
The paper's Eq. (3)-(6) global-memory volumes describe its own
C-split kernel and are reported alongside for contrast (paper_volumes()).
"""
from __future__ import annotations

import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# Nominal B200 facts (B200_PROFILING.md): 148 SMs, clocks.max.sm 1965 MHz.
SMS = 148
FP32_LANES_PER_SM = 128          # FFMA lanes per SM (4 SMSPs x 32)
SM_MAX_MHZ_NOMINAL = 1965.0
FALLBACK_HBM_GBS = 6650.0        # profiling guide fallback
FALLBACK_BF16_TFLOPS = 1590.0
TF32_OVER_BF16 = 1.1 / 2.25      # nominal dense ratio (guide table)


def out_dim(h: int, k: int, s: int, p: int) -> int:
    return (h + 2 * p - k) // s + 1


def stage_flops(H, W, C, N, D1, D2, K, stride=1, pad=None, B=1):
    pad = (K - 1) // 2 if pad is None else pad
    Ho, Wo = out_dim(H, K, stride, pad), out_dim(W, K, stride, pad)
    return (2 * B * H * W * C * D1, 2 * B * Ho * Wo * D1 * D2 * K * K, 2 * B * Ho * Wo * D2 * N)


def tkd_flops(shape, B=None) -> int:
    B = shape.B if B is None else B
    return sum(stage_flops(shape.H, shape.W, shape.C, shape.N, shape.D1, shape.D2, shape.K,
                           shape.stride, shape.pad, B))


def dense_flops(shape, B=None) -> int:
    """The uncompressed K x K conv the TKD layer replaces (S:L440 'orig')."""
    B = shape.B if B is None else B
    return 2 * B * shape.Ho * shape.Wo * shape.C * shape.N * shape.K * shape.K


def weight_bytes(shape, bias=False) -> int:
    return 4 * (shape.C * shape.D1 + shape.D1 * shape.D2 * shape.K * shape.K
                + shape.D2 * shape.N + (shape.N if bias else 0))


def tkd_bytes(shape, B=None, bias=False) -> int:
    """Fused algorithmic HBM bytes: input once, output once, weights once."""
    B = shape.B if B is None else B
    return 4 * B * (shape.H * shape.W * shape.C + shape.Ho * shape.Wo * shape.N) \
        + weight_bytes(shape, bias)


def paper_volumes(shape, TH, TW, TC):
    """Eqs. (3)-(5) of the paper for the core conv alone, in elements,
    with the core's channels C=D1, N=D2 (the listing only sees the core conv)."""
    from math import ceil
    H, W, C, N, R, S = shape.H, shape.W, shape.D1, shape.D2, shape.K, shape.K
    vk = ceil(H / TH) * ceil(W / TW) * C * N
    vx = ceil(H / TH) * ceil(W / TW) * C * (TH + R - 1) * (TW + S - 1)
    vy = H * W * N * C // TC
    return vk, vx, vy, vk + vx + vy


def measured_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        return {"hbm_gbs": float(m["hbm_gbs"]), "bf16_tflops": float(m["bf16_tflops"]),
                "bf16_tflops_sustained": float(m.get("bf16_tflops_sustained", m["bf16_tflops"])),
                "sm_max_mhz": float(m.get("sm_max_mhz", SM_MAX_MHZ_NOMINAL)),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": FALLBACK_HBM_GBS, "bf16_tflops": FALLBACK_BF16_TFLOPS,
            "bf16_tflops_sustained": 1400.0, "sm_max_mhz": SM_MAX_MHZ_NOMINAL,
            "source": "fallback (B200_PROFILING.md)"}


def fp32_alu_tflops(sm_mhz: float | None = None) -> float:
    """FFMA peak: 148 SMs x 128 lanes x 2 FLOP x clock."""
    mhz = SM_MAX_MHZ_NOMINAL if sm_mhz is None else sm_mhz
    return SMS * FP32_LANES_PER_SM * 2 * mhz * 1e6 / 1e12


def engine_peak_tflops(math: str, peaks: dict | None = None) -> float:
    peaks = peaks or measured_peaks()
    if math == "fp32":
        return fp32_alu_tflops(peaks["sm_max_mhz"])
    if math == "3xbf16":  # three bf16 products per fp32-grade product
        return peaks["bf16_tflops"] / 3.0
    tf32 = peaks["bf16_tflops"] * TF32_OVER_BF16
    return tf32 if math == "tf32" else tf32 / 3.0
