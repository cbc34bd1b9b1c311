"""Hardware-aware rank selection (paper_2211_03715_b200/ranksel.py): FLOP accounting
pinned to SPEC's hand-derived example, and the selection's invariants
checked against independent re-summation and brute force on synthetic tables."""
import itertools
import random

import pytest

from paper_2211_03715_b200 import ranksel
from paper_2211_03715_b200.ranksel import LayerSpec


def test_flops_counts_spec_example():
    # 14x14, C=N=256, 3x3, d1=d2=64 -> orig 231,211,008; tucker 27,295,744
    orig, tk = ranksel.flops_counts(14, 14, 256, 256, 3, 1, 1, 64, 64)
    assert orig == 231_211_008
    assert tk == 6_422_528 + 14_450_688 + 6_422_528 == 27_295_744


def test_flops_counts_pointwise_overhead_and_bounds():
    # d1 = C, d2 = N on a 1x1 layer: the factorisation costs more than the dense layer
    orig, tk = ranksel.flops_counts(8, 8, 16, 16, 1, 1, 0, 16, 16)
    assert tk > orig
    for bad in ((0, 4), (4, 0), (17, 4), (4, 17)):
        with pytest.raises(ValueError):
            ranksel.flops_counts(8, 8, 16, 16, 3, 1, 1, *bad)


def test_default_grid_multiples_of_eighth():
    g = ranksel.default_grid(64, 128)
    assert sorted({a for a, _ in g}) == [8, 16, 24, 32, 40, 48, 56, 64]
    assert sorted({b for _, b in g}) == [16, 32, 48, 64, 80, 96, 112, 128]
    assert len(g) == 64
    assert len(ranksel.default_grid(64, 128, ranksel.HALF_GRID)) == 16


def synthetic_tables(layers, seed=0, jitter=0.3):
    """Latency = a + b * tucker FLOPs, plus a non-monotone per-point jitter (as measured
    tables are: padding to tensor-core tiles makes some smaller ranks slower)."""
    rng = random.Random(seed)
    tabs = {}
    for l in layers:
        tabs[l.name] = {}
        for r in ranksel.default_grid(l.C, l.N, ranksel.HALF_GRID):
            f = l.flops(*r)[1]
            tabs[l.name][r] = 5.0 + f / 2e7 * (1.0 + jitter * rng.random())
    return tabs


SLACK = 0.05


def resum(layers, ranks):
    tk = sum(l.count * l.flops(*ranks[l.name])[1] for l in layers)
    orig = sum(l.count * l.flops(*ranks[l.name])[0] for l in layers)
    return 1.0 - tk / orig


def test_tiny_budget_keeps_max_ranks():
    layers = ranksel.resnet18_layers()
    tabs = synthetic_tables(layers)
    plan = ranksel.select_ranks(layers, tabs, 1e-6, slack=1e-6)
    # only the grid's largest ranks remove no FLOPs at all... none of them does here, so
    # the plan is the least-reducing one the grid allows, and it is infeasible
    assert not plan.feasible
    assert all(plan.ranks[l.name] == max(tabs[l.name]) for l in layers)


def test_forced_single_layer_move():
    l = LayerSpec("one", 8, 8, 16, 16, 3, 1, 1, 1)
    tabs = {"one": {(2, 2): 1.0, (4, 4): 2.0}}
    o, t22 = l.flops(2, 2)
    _, t44 = l.flops(4, 4)
    budget = 1.0 - (t22 + t44) / 2 / o   # only (2, 2) satisfies it
    plan = ranksel.select_ranks([l], tabs, budget, slack=0.5)
    assert plan.ranks["one"] == (2, 2) and plan.feasible


@pytest.mark.parametrize("budget", [0.63, 0.7, 0.8, 0.9])
def test_resnet18_budget_invariants(budget):
    layers = ranksel.resnet18_layers()
    tabs = synthetic_tables(layers, seed=int(budget * 100))
    plan = ranksel.select_ranks(layers, tabs, budget, SLACK)
    assert plan.feasible
    # achieved reduction re-verified by independent re-summation: inside [B, B + slack]
    assert budget - 1e-9 <= resum(layers, plan.ranks) <= budget + SLACK + 1e-9
    assert abs(resum(layers, plan.ranks) - plan.reduction) < 1e-9
    for l in layers:
        a, b = plan.ranks[l.name]
        assert 1 <= a <= l.C and 1 <= b <= l.N and (a, b) in tabs[l.name]
    # determinism
    assert ranksel.select_ranks(layers, tabs, budget, SLACK).ranks == plan.ranks
    # local optimality: no single-layer change inside the band lowers the latency
    for l in layers:
        for r in tabs[l.name]:
            trial = dict(plan.ranks)
            trial[l.name] = r
            if budget - 1e-9 <= resum(layers, trial) <= budget + SLACK + 1e-9:
                lat = sum(x.count * tabs[x.name][trial[x.name]] for x in layers)
                assert lat >= plan.latency_us - 1e-6
    # the exact optimum is never worse than the greedy plan
    exact = ranksel.select_ranks_exact(layers, tabs, budget, SLACK)
    assert exact.feasible and exact.latency_us <= plan.latency_us + 1e-6
    assert budget - 1e-9 <= resum(layers, exact.ranks) <= budget + SLACK + 1e-9


def test_exact_matches_brute_force():
    layers = [LayerSpec("a", 14, 14, 64, 64, 3, 1, 1, 2), LayerSpec("b", 7, 7, 128, 64, 3, 2, 1, 1),
              LayerSpec("c", 28, 28, 32, 32, 3, 1, 1, 3)]
    tabs = synthetic_tables(layers, seed=7, jitter=0.8)
    for budget in (0.3, 0.6, 0.75, 0.85):
        best = None
        for combo in itertools.product(*[sorted(tabs[l.name]) for l in layers]):
            ranks = {l.name: r for l, r in zip(layers, combo)}
            if not budget - 1e-9 <= resum(layers, ranks) <= budget + SLACK + 1e-9:
                continue
            lat = sum(l.count * tabs[l.name][ranks[l.name]] for l in layers)
            if best is None or lat < best - 1e-9:
                best = lat
        exact = ranksel.select_ranks_exact(layers, tabs, budget, SLACK)
        if best is None:
            assert not exact.feasible
        else:
            assert exact.feasible and abs(exact.latency_us - best) < 1e-6


def test_infeasible_budget_reports_max_reduction():
    layers = ranksel.resnet18_layers()
    tabs = synthetic_tables(layers)
    plan = ranksel.select_ranks(layers, tabs, 0.99)
    assert not plan.feasible
    # it went all the way down: the reported reduction is the largest achievable on the grid
    smallest = {l.name: min(tabs[l.name], key=lambda r: l.flops(*r)[1]) for l in layers}
    assert abs(plan.reduction - resum(layers, smallest)) < 1e-9


def test_bad_inputs():
    layers = ranksel.resnet18_layers()
    tabs = synthetic_tables(layers)
    for b in (0.0, 1.0, -0.1):
        with pytest.raises(ValueError):
            ranksel.select_ranks(layers, tabs, b)
    with pytest.raises(ValueError):
        ranksel.select_ranks(layers, {k: v for k, v in list(tabs.items())[:-1]}, 0.5)


def test_table_json_round_trip():
    l = ranksel.resnet18_layers()[0]
    tab = {(8, 8): 10.0, (16, 32): 12.5}
    obj = ranksel.table_to_json(l, tab, 32, "3xbf16")
    l2, tab2 = ranksel.table_from_json(obj)
    assert l2 == l and tab2 == tab
    assert obj["rows"][0]["tucker_flops"] == 32 * l.flops(8, 8)[1]


@pytest.mark.gpu
def test_measured_table_through_the_c_abi():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    l = LayerSpec("t", 14, 14, 64, 64, 3, 1, 1, 1)
    tab = ranksel.measure_table(l, [(8, 8), (32, 32)], batch=4, math_mode="3xbf16", iters=5)
    assert set(tab) == {(8, 8), (32, 32)} and all(0 < v < 1e5 for v in tab.values())
