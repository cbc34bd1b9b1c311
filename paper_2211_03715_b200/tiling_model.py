"""The paper's analytical tiling model (Eqs. 1-6) and its re-fit to B200
(SURVEY §8(f) NEXT-3).

Part A -- the model as the paper states it, for its own core-convolution kernel
(thread block = TH x TW output pixels x TC input channels, N threads, fp32 FFMA):

  num_blks  = ceil(H/TH) ceil(W/TW) ceil(C/TC);  Num_ths = num_blks * N
  comp_latency_blk = 2 (TH+R-1)(TW+S-1) TC GPU_ths R S / GPU_peak
  comp_waves = ceil(Num_ths / (GPU_ths * Occupancy))                         Eq. (1)
  comp_latency = comp_waves * comp_latency_blk                                 Eq. (2)
  volume_k = ceil(H/TH) ceil(W/TW) C N                                         Eq. (3)
  volume_x = ceil(H/TH) ceil(W/TW) C (TH+R-1)(TW+S-1)                          Eq. (4)
  volume_y = H W N C/TC                                                        Eq. (5)
  volume_total = volume_x + volume_k + volume_y                                Eq. (6)
  selection: sort by comp_latency, keep the top fraction, pick min memory latency

Occupancy (not defined by the paper beyond "estimated by the hardware metrics such as
shared memory size") and the ceilings on ragged tiles follow SPEC's readings
(S:L215-220); the SPEC worked values pin every function (tests/golden/
paper_model_spec.json: S:L220).

Part B -- the same structure re-fitted to this implementation on B200: every kernel of
a 3xBF16 plan is a persistent grid over 148 SMs, so its latency is
  waves * per-tile latency  (Eqs. 1-2 with the per-tile MMA issue cost measured on B200,
                             DESIGN.md §8, times an in-situ factor kappa)
and its memory term is the global-memory volume of the variant (Eqs. 3-6's role: X, the
X'/Z intermediates the unfused variants round-trip, Y, the weights) over the measured
HBM bandwidth, plus a fixed per-launch cost L0; kappa and L0 are fitted to the measured
exhaustive search (scripts/tiling_search_r18.py).  The two-stage selection is the
paper's: candidates sorted by the compute term, the top fraction kept, the one with the
least memory time chosen.
"""
from __future__ import annotations

import dataclasses
import itertools
import math
from typing import Dict, Iterable, List, Optional, Sequence, Tuple


# ============================================================ Part A: the paper's model
@dataclasses.dataclass(frozen=True)
class GpuSpec:
    name: str
    num_sms: int
    max_threads_per_sm: int
    max_threads_per_block: int
    smem_per_block: int
    smem_per_sm: int
    max_blocks_per_sm: int
    peak_flops: float          # FP32, FMA = 2 FLOPs
    mem_bandwidth: float       # bytes/s
    bandwidth_efficiency: float = 0.8
    top_frac: float = 0.05

    @property
    def gpu_ths(self) -> int:
        return self.num_sms * self.max_threads_per_sm


# B200 (sm_100a): 148 SMs, 2048 threads and 228 KB shared memory per SM, 227 KB per
# block (opt-in), 32 blocks/SM; FP32 FFMA peak 148 x 128 x 2 x 1.965 GHz; HBM from
# MEASURED_PEAKS.json when present (roofline.measured_peaks), else the guide's fallback.
def b200_spec(hbm_gbs: Optional[float] = None) -> GpuSpec:
    if hbm_gbs is None:
        from . import roofline
        hbm_gbs = roofline.measured_peaks()["hbm_gbs"]
    return GpuSpec("b200", 148, 2048, 1024, 232448, 233472, 32, 148 * 128 * 2 * 1.965e9, hbm_gbs * 1e9)


def estimate_occupancy(R: int, S: int, TH: int, TW: int, TC: int, N: int, g: GpuSpec) -> Tuple[float, bool]:
    """(occupancy, valid): smem_blk = TC (TH+R-1)(TW+S-1) 4 bytes."""
    smem_blk = TC * (TH + R - 1) * (TW + S - 1) * 4
    if smem_blk > g.smem_per_block or N > g.max_threads_per_block or smem_blk <= 0:
        return 0.0, False
    blocks = min(g.smem_per_sm // smem_blk, g.max_blocks_per_sm, g.max_threads_per_sm // N)
    if blocks < 1:
        return 0.0, False
    return min(1.0, max(blocks * N / g.max_threads_per_sm, 1e-9)), True


def comp_latency_block(R: int, S: int, TH: int, TW: int, TC: int, g: GpuSpec) -> float:
    """The paper's closed form (N cancels), seconds."""
    return 2.0 * (TH + R - 1) * (TW + S - 1) * TC * g.gpu_ths * R * S / g.peak_flops


def comp_waves(H: int, W: int, C: int, N: int, TH: int, TW: int, TC: int, g: GpuSpec, occupancy: float) -> int:
    """Eq. (1) with ceilings on the tile counts."""
    num_ths = math.ceil(H / TH) * math.ceil(W / TW) * math.ceil(C / TC) * N
    return max(1, math.ceil(num_ths / (g.gpu_ths * occupancy)))


def comp_latency(H, W, C, N, R, S, TH, TW, TC, g: GpuSpec) -> Optional[float]:
    """Eq. (2); None for an invalid tiling."""
    occ, ok = estimate_occupancy(R, S, TH, TW, TC, N, g)
    if not ok:
        return None
    return comp_waves(H, W, C, N, TH, TW, TC, g, occ) * comp_latency_block(R, S, TH, TW, TC, g)


def data_volumes(H, W, C, N, R, S, TH, TW, TC) -> Tuple[int, int, int, int]:
    """Eqs. (3)-(6), elements (ceiling on C/TC for ragged channel tiles)."""
    tiles = math.ceil(H / TH) * math.ceil(W / TW)
    vk = tiles * C * N
    vx = tiles * C * (TH + R - 1) * (TW + S - 1)
    vy = H * W * N * math.ceil(C / TC)
    return vk, vx, vy, vx + vk + vy


def mem_latency(total_volume: int, g: GpuSpec) -> float:
    return total_volume * 4 / (g.mem_bandwidth * g.bandwidth_efficiency)


def enumerate_tilings(H, W, C, R, S, N, g: GpuSpec, divisors_only: bool = False) -> List[Tuple[int, int, int]]:
    """Every valid (TH, TW, TC), lexicographic."""
    def rng(n):
        return [d for d in range(1, n + 1) if n % d == 0] if divisors_only else range(1, n + 1)
    out = []
    for th in rng(H):
        for tw in rng(W):
            for tc in rng(C):
                if estimate_occupancy(R, S, th, tw, tc, N, g)[1]:
                    out.append((th, tw, tc))
    return out


def select_tiling_analytical(H, W, C, N, R, S, g: GpuSpec, divisors_only: bool = False):
    """The paper's two-stage selection: sort by comp_latency, keep the top
    fraction (at least one), pick the minimum memory latency; ties lexicographic."""
    cands = enumerate_tilings(H, W, C, R, S, N, g, divisors_only)
    if not cands:
        raise ValueError("no valid tiling")
    scored = sorted((comp_latency(H, W, C, N, R, S, *t, g), t) for t in cands)
    keep = scored[:max(1, int(math.ceil(len(scored) * g.top_frac)))]
    best = min(keep, key=lambda ct: (mem_latency(data_volumes(H, W, C, N, R, S, *ct[1])[3], g), ct[1]))
    return best[1]


# ====================================================== Part B: the B200 re-fit (3xBF16)
HINT_SPACE = {
    "fused_layer": (1, 0),           # the single-launch layer kernel when it fits / never
    "core3": (-1, 0),                # stage 3 fused into the core kernel when it fits / never
    "bn_stage1": (32, 64, 128),
    "bn_core": (32, 64, 128),
    "bn_stage3": (32, 64, 128),
    "gsplit_core": (1, 2, 4),
}


def hint_points(space: Dict[str, Sequence[int]] = HINT_SPACE) -> List[Dict[str, int]]:
    keys = list(space)
    return [dict(zip(keys, v)) for v in itertools.product(*(space[k] for k in keys))]


def _r(v, m):
    return (v + m - 1) // m * m


def mma_cycles(n: int) -> float:
    """Isolated tcgen05.mma kind::f16 M=128 K=16 issue cost on B200 (DESIGN.md §8,
    scripts/mma_microbench4.cu): a ~45-cycle floor below N = 96, N/2 above."""
    return max(44.8, n / 2.0)


@dataclasses.dataclass
class LayerGeom:
    B: int
    C: int
    N: int
    H: int
    W: int
    D1: int
    D2: int
    K: int = 3
    s: int = 1
    p: int = 1

    @property
    def Ho(self):
        return (self.H + 2 * self.p - self.K) // self.s + 1

    @property
    def Wo(self):
        return (self.W + 2 * self.p - self.K) // self.s + 1


def fused_layer_eligible(L: LayerGeom) -> bool:
    """Mirror of tdc_api.cu plan_layer's shape conditions (not its shared-memory fit)."""
    Wp = L.W + 2 * L.p
    return (L.s == 1 and L.C % 4 == 0 and _r(L.D1, 32) <= 128 and _r(L.D2, 32) <= 128 and _r(L.N, 32) <= 128
            and Wp <= 128 and 2 * _r(L.D1, 32) * 2 + 4 * _r(L.D2, 32) + 4 * _r(L.N, 32) <= 512)


def kernels_of(L: LayerGeom, h: Dict[str, int], num_sms: int = 148) -> List[dict]:
    """The kernels a hint point launches: tiles, MMA cycles per tile (isolated rates),
    global bytes.  Geometry as in tdc_api.cu (phase grid for the core)."""
    D1s, D2s, N3p = _r(L.D1, 32), _r(L.D2, 32), _r(L.N, 32)
    C64, D2p = _r(L.C, 64), _r(L.D2, 64)
    M1, M3 = L.B * L.H * L.W, L.B * L.Ho * L.Wo
    Hq, Wq = -(-(L.H + 2 * L.p) // L.s), -(-(L.W + 2 * L.p) // L.s)
    M2 = L.B * Hq * Wq
    KK = L.K * L.K
    x_b, y_b = 4 * M1 * L.C, 4 * M3 * L.N
    w_b = 4 * (L.C * L.D1 + L.D1 * L.D2 * KK + L.D2 * L.N)
    others = any(h.get(k, 0) > 0 for k in ("bn_stage1", "bn_core", "bn_stage3", "gsplit_core")) or h.get("core3", -1) == 0
    fl = h.get("fused_layer", -1)
    if fused_layer_eligible(L) and (fl == 1 or (fl == -1 and not others)):  # as tdc_api.cu plan_layer
        R = max(1, min(128 // (L.W + 2 * L.p), L.Ho))
        tiles = L.B * -(-L.Ho // R)
        cyc = ((C64 // 16) * (mma_cycles(2 * D1s) + mma_cycles(D1s)) * 1.0 +
               KK * (D1s // 16) * (mma_cycles(2 * D2s) + mma_cycles(D2s)) +
               (D2s // 16) * (mma_cycles(2 * N3p) + mma_cycles(N3p)))
        return [{"name": "layer", "tiles": tiles, "cyc": cyc, "bytes": x_b + y_b + w_b}]
    bn1, bn2, bn3, gs = h.get("bn_stage1", 64) or 64, h.get("bn_core", 64) or 64, h.get("bn_stage3", 64) or 64, \
        max(1, h.get("gsplit_core", 1))
    xg_b = 2 * 2 * M2 * L.s * L.s * D1s          # X' hi/lo bf16 phase grid, written and read
    ks = [{"name": "stage1", "tiles": -(-M1 // 128) * -(-D1s // bn1), "cyc": (C64 // 16) * 3 * mma_cycles(bn1),
           "bytes": x_b + xg_b}]
    core3 = h.get("core3", -1) != 0 and D2s <= 128 and 2 * N3p <= 256
    ncat = 2 * bn2 <= 128
    core_cyc = KK * (D1s // 16) * (2 * mma_cycles(2 * bn2) if ncat else 3 * mma_cycles(bn2)) / gs
    if core3:
        core_cyc = KK * (D1s // 16) * (mma_cycles(2 * D2s) + mma_cycles(D2s)) + \
            (D2s // 16) * (mma_cycles(2 * N3p) + mma_cycles(N3p))
        ks.append({"name": "core3", "tiles": -(-M2 // 128), "cyc": core_cyc, "bytes": xg_b + y_b})
    else:
        z_b = 2 * 2 * M3 * D2p
        ks.append({"name": "core", "tiles": -(-M2 // 128) * -(-D2s // bn2) * gs, "cyc": core_cyc,
                   "bytes": xg_b + z_b + (gs - 1) * 8 * M2 * D2s})
        ks.append({"name": "stage3", "tiles": -(-M3 // 128) * -(-L.N // bn3), "cyc": (D2p // 16) * 3 * mma_cycles(bn3),
                   "bytes": z_b + y_b})
    ks[0]["bytes"] += w_b
    return ks


@dataclasses.dataclass
class Refit:
    """B200 constants of Part B: in-situ MMA factor kappa, fixed cost per launch (s),
    SM clock, HBM bandwidth (bytes/s)."""
    kappa: float = 1.8
    l0: float = 4e-6
    clock_hz: float = 1.965e9
    hbm: float = 6.5e12
    num_sms: int = 148

    def comp(self, ks: List[dict]) -> float:
        return sum(math.ceil(k["tiles"] / self.num_sms) * k["cyc"] * self.kappa / self.clock_hz for k in ks)

    def mem(self, ks: List[dict]) -> float:
        return sum(k["bytes"] for k in ks) / self.hbm

    def predict(self, ks: List[dict]) -> float:
        return sum(self.l0 + max(math.ceil(k["tiles"] / self.num_sms) * k["cyc"] * self.kappa / self.clock_hz,
                                 k["bytes"] / self.hbm) for k in ks)


def select_hints_analytical(L: LayerGeom, fit: Refit, points: Optional[Iterable[Dict[str, int]]] = None,
                            top_frac: float = 0.15) -> Dict[str, int]:
    """The paper's two-stage rule on the re-fitted terms: sort the candidate kernel plans by
    compute latency (waves x per-tile MMA cost, + L0 per launch), keep the top fraction,
    pick the least memory time; ties by the full prediction, then the hint order."""
    pts = list(points) if points is not None else hint_points()
    scored = []
    for i, h in enumerate(pts):
        ks = kernels_of(L, h)
        scored.append((fit.comp(ks) + fit.l0 * len(ks), i, h, ks))
    scored.sort(key=lambda t: (t[0], t[1]))
    keep = scored[:max(1, int(math.ceil(len(scored) * top_frac)))]
    best = min(keep, key=lambda t: (fit.mem(t[3]) + fit.l0 * len(t[3]), fit.predict(t[3]), t[1]))
    return dict(best[2])


def fit_refit(samples: Sequence[Tuple[LayerGeom, Dict[str, int], float]], hbm: Optional[float] = None) -> Refit:
    """Least squares (in log time) of kappa and L0 over measured (layer, hints, seconds)."""
    base = Refit() if hbm is None else Refit(hbm=hbm)
    best, best_err = base, float("inf")
    for kappa in [1.0 + 0.05 * i for i in range(41)]:           # 1.0 .. 3.0
        for l0 in [0.5e-6 * i for i in range(1, 25)]:           # 0.5 .. 12 us
            f = dataclasses.replace(base, kappa=kappa, l0=l0)
            err = sum((math.log(f.predict(kernels_of(L, h))) - math.log(t)) ** 2 for L, h, t in samples)
            if err < best_err:
                best, best_err = f, err
    return best
