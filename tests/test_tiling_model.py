"""The paper's analytical tiling model (Eqs. 1-6) pinned to SPEC's hand-
evaluated worked values and to the properties the
equations imply; and the structure of the B200 re-fit (NEXT-3)."""
import math

from paper_2211_03715_b200 import tiling_model as tm

A100_LIKE = tm.GpuSpec("a100-like", 108, 2048, 1024, 49152, 167936, 32, 19.5e12, 1.555e12)


def test_occupancy_worked_example(golden):
    g = golden("paper_model_spec.json")["occupancy"]
    spec = tm.GpuSpec("x", 108, g["threads_per_sm"], 1024, g["smem_per_block"], g["smem_per_sm"],
                      g["max_blocks_per_sm"], 19.5e12, 1.555e12)
    occ, ok = tm.estimate_occupancy(g["R"], g["S"], g["TH"], g["TW"], g["TC"], g["N"], spec)
    assert ok and occ == g["occupancy"]
    assert g["TC"] * (g["TH"] + 2) * (g["TW"] + 2) * 4 == g["smem_blk"]
    # trivial cases: saturating block, smem overflow
    import dataclasses
    big = dataclasses.replace(spec, max_threads_per_block=2048)          # a block may fill the SM
    assert tm.estimate_occupancy(1, 1, 1, 1, 1, 2048, big) == (1.0, True)
    assert tm.estimate_occupancy(3, 3, 64, 64, 64, 64, spec)[1] is False


def test_comp_latency_block_and_waves(golden):
    g = golden("paper_model_spec.json")
    c = g["comp_latency_block"]
    spec = tm.GpuSpec("x", 108, 2048, 1024, 49152, 167936, 32, c["peak_flops"], 1.555e12)
    assert spec.gpu_ths == c["gpu_ths"]
    t = tm.comp_latency_block(c["R"], c["S"], c["TH"], c["TW"], c["TC"], spec)
    assert abs(t - c["seconds"]) <= c["rel_tol"] * c["seconds"]
    assert tm.comp_latency_block(3, 3, 8, 8, 32, spec) == 2 * t            # linear in TC
    assert tm.comp_latency_block(1, 1, 1, 1, 1, spec) == 2 * spec.gpu_ths / spec.peak_flops
    w = g["comp_waves"]                               # S:L236, Eq. (1)
    assert 7 * 7 * 4 * 64 == w["num_ths"]
    assert tm.comp_waves(w["H"], w["W"], w["C"], w["N"], w["TH"], w["TW"], w["TC"], spec, w["occupancy"]) == w["waves"]
    # ceiling step: exactly GPU_ths threads -> 1 wave, one more -> 2
    assert tm.comp_waves(108, 1, 2048, 1, 1, 1, 1, spec, 1.0) == 1
    assert tm.comp_waves(108 * 2048 + 1, 1, 1, 1, 1, 1, 1, spec, 1.0) == 2


def test_volumes_worked_example_and_structure(golden):
    g = golden("paper_model_spec.json")["volumes"]   # S:L250, Eqs. (3)-(6)
    vk, vx, vy, tot = tm.data_volumes(g["H"], g["W"], g["C"], g["N"], g["R"], g["S"], g["TH"], g["TW"], g["TC"])
    assert (vk, vx, vy, tot) == (g["vk"], g["vx"], g["vy"], g["total"])
    # single-tile reduction and independence properties
    assert tm.data_volumes(14, 14, 32, 16, 3, 3, 14, 14, 32)[:3] == (32 * 16, 32 * 16 * 16, 14 * 14 * 16)
    assert tm.data_volumes(14, 14, 32, 16, 3, 3, 7, 7, 8)[2] == tm.data_volumes(14, 14, 32, 16, 3, 3, 2, 2, 8)[2]
    assert tm.data_volumes(14, 14, 32, 16, 3, 3, 7, 7, 8)[0] == tm.data_volumes(14, 14, 32, 16, 3, 3, 7, 7, 32)[0]
    for th in range(1, 14):  # vk non-increasing in TH; vy non-increasing in TC
        assert tm.data_volumes(14, 14, 8, 8, 3, 3, th + 1, 4, 2)[0] <= tm.data_volumes(14, 14, 8, 8, 3, 3, th, 4, 2)[0]
    for tc in range(1, 8):
        assert tm.data_volumes(14, 14, 8, 8, 3, 3, 4, 4, tc + 1)[2] <= tm.data_volumes(14, 14, 8, 8, 3, 3, 4, 4, tc)[2]


def test_mem_latency_examples():
    spec = tm.GpuSpec("x", 108, 2048, 1024, 49152, 167936, 32, 19.5e12, 1.555e12)
    assert tm.mem_latency(0, spec) == 0
    assert abs(tm.mem_latency(10 ** 9, spec) - 3.215e-3) < 1e-6
    half = tm.GpuSpec("x", 108, 2048, 1024, 49152, 167936, 32, 19.5e12, 1.555e12, bandwidth_efficiency=0.4)
    assert abs(tm.mem_latency(10 ** 6, half) - 2 * tm.mem_latency(10 ** 6, spec)) < 1e-15


def test_analytical_selection_against_exhaustive_recomputation():
    """the returned tiling is in the top fraction by comp latency and has the least
    memory latency among those, verified by recomputing every candidate."""
    H = W = 14
    C = N = 16
    spec = A100_LIKE
    th, tw, tc = tm.select_tiling_analytical(H, W, C, N, 3, 3, spec)
    cands = tm.enumerate_tilings(H, W, C, 3, 3, N, spec)
    assert (th, tw, tc) in cands
    comps = sorted(tm.comp_latency(H, W, C, N, 3, 3, *t, spec) for t in cands)
    k = max(1, math.ceil(len(comps) * spec.top_frac))
    mine = tm.comp_latency(H, W, C, N, 3, 3, th, tw, tc, spec)
    assert mine <= comps[k - 1]
    kept = [t for t in cands if tm.comp_latency(H, W, C, N, 3, 3, *t, spec) <= comps[k - 1]]
    assert min(tm.data_volumes(H, W, C, N, 3, 3, *t)[3] for t in kept) == tm.data_volumes(H, W, C, N, 3, 3, th, tw, tc)[3]
    # scaling peak and bandwidth together leaves the choice unchanged
    import dataclasses
    s2 = dataclasses.replace(spec, peak_flops=spec.peak_flops * 3, mem_bandwidth=spec.mem_bandwidth * 3)
    assert tm.select_tiling_analytical(H, W, C, N, 3, 3, s2) == (th, tw, tc)


def test_b200_refit_structure():
    L = tm.LayerGeom(32, 64, 64, 56, 56, 32, 32)
    pts = tm.hint_points()
    assert len(pts) == 2 * 2 * 3 * 3 * 3 * 3
    fused = tm.kernels_of(L, {"fused_layer": 1, "core3": -1, "bn_stage1": 64, "bn_core": 0, "bn_stage3": 0})
    assert tm.kernels_of(L, {"fused_layer": -1})[0]["name"] == "layer"
    three = tm.kernels_of(L, {"fused_layer": 0, "core3": 0, "bn_stage1": 64, "bn_core": 64, "bn_stage3": 64})
    assert [k["name"] for k in fused] == ["layer"] and [k["name"] for k in three] == ["stage1", "core", "stage3"]
    # the fused plan moves exactly the algorithmic bytes; the unfused ones round-trip X' and Z
    from paper_2211_03715_b200 import roofline
    import synth
    assert fused[0]["bytes"] == roofline.tkd_bytes(synth.LayerShape(32, 64, 64, 56, 56, 32, 32))
    assert sum(k["bytes"] for k in three) > fused[0]["bytes"]
    fit = tm.Refit()
    h = tm.select_hints_analytical(L, fit)
    assert h in pts
    # fitting recovers the constants that generated synthetic samples
    truth = tm.Refit(kappa=1.6, l0=3e-6)
    samples = [(L, p, truth.predict(tm.kernels_of(L, p))) for p in pts[::7]]
    f = tm.fit_refit(samples)
    assert abs(f.kappa - 1.6) < 0.06 and abs(f.l0 - 3e-6) < 0.6e-6
