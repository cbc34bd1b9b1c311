"""Measured autotune of the 3xBF16 layer planner.

The paper picks tile sizes with an analytical model of waves, occupancy and global
volumes (Eqs. 1-6) and reports a ~25 % gap to an exhaustive search.  Here
the planner is a set of B200 heuristics (N tiles from the parallelism
rule and the shared-memory fit, core3 fusion when D2 fits one tile, split-K opt-in);
this module measures the alternatives through the C-ABI planner overrides
(``tdc_conv_plan_ex`` hints) and reports the planner's gap to the best found.

Search: coordinate descent over the knobs (each knob swept with the others held at
the current best, two passes), starting from the planner's own choice -- the full
cross product (~10^3 points per layer) is not worth a GPU-minute each.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Dict, List, Optional

KNOBS = {
    "core3": [-1, 0],
    "bn_core": [0, 32, 64, 128, 256],
    "bn_stage1": [0, 32, 64, 128],
    "bn_stage3": [0, 32, 64, 128, 256],
    "ksplit_core": [0, 1, 2, 3, 4],
    "ksplit_stage1": [0, 1, 2],
}


@dataclasses.dataclass
class TuneResult:
    planner_us: float
    best_us: float
    best_hints: Dict[str, int]
    measured: int
    trials: List[tuple]

    @property
    def gap(self) -> float:
        """planner time / best time - 1 (0 = the planner found the best point)."""
        return self.planner_us / self.best_us - 1.0


def coordinate_descent(measure: Callable[[Dict[str, int]], Optional[float]], knobs=KNOBS, passes: int = 2,
                       start: Optional[Dict[str, int]] = None) -> TuneResult:
    """`measure(hints) -> µs` (None if the point is invalid).  Deterministic: knobs in
    the given order, values in the given order, ties keep the earlier point."""
    cache: Dict[tuple, Optional[float]] = {}

    def m(h):
        key = tuple(sorted(h.items()))
        if key not in cache:
            cache[key] = measure(dict(h))
        return cache[key]

    cur = dict(start or {k: v[0] for k, v in knobs.items()})
    base = m(cur)
    if base is None:
        raise ValueError("the starting point (planner default) must be measurable")
    best_t = base
    for _ in range(passes):
        improved = False
        for k, vals in knobs.items():
            for v in vals:
                if v == cur[k]:
                    continue
                trial = dict(cur)
                trial[k] = v
                t = m(trial)
                if t is not None and t < best_t - 1e-9:
                    best_t, cur, improved = t, trial, True
        if not improved:
            break
    trials = [(dict(k), t) for k, t in cache.items()]
    return TuneResult(base, best_t, cur, len(cache), trials)


def measure_hints_us(shape, hints: Dict[str, int], iters: int = 30, seed: int = 42) -> Optional[float]:
    """Mean µs per forward of a 3xBF16 layer planned with `hints` (back-to-back forwards,
    CUDA events, inputs rotated over > 2x L2)."""
    import torch

    import synth
    from . import tdc

    d = synth.make_layer(shape, seed=seed)
    try:
        plan = tdc.ConvPlan(shape, d, math=tdc.TDC_MATH_3XBF16, hints=dict(hints))
    except tdc.TdcError:
        return None
    try:
        ws = 4 * (shape.B * shape.H * shape.W * shape.C + shape.B * shape.Ho * shape.Wo * shape.N)
        nbuf = max(2, -(-2 * 126 * 2 ** 20 // ws))
        x0 = torch.from_numpy(synth.nchw_to_nhwc(d["x"])).cuda()
        xs = [x0] + [x0.clone() for _ in range(nbuf - 1)]
        ys = [torch.empty((shape.B, shape.Ho, shape.Wo, shape.N), device="cuda") for _ in range(nbuf)]
        st = torch.cuda.current_stream()
        for k in range(nbuf):
            plan.forward(xs[k], ys[k])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for k in range(iters):
            plan.forward(xs[k % nbuf], ys[k % nbuf])
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / iters
    finally:
        plan.close()
