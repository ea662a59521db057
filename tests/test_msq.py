"""Fusion-aware MSQ: the oracle's brute force pinned by closed forms, and the
library's exact Pareto-frontier solver (qp_plan_msq, host-only) against the brute force."""
import math

import numpy as np
import pytest

from oracle import msq as M
from paper_2509_20214_b200 import _lib as QL


def test_partition_counts():
    # {q,k,v}: Bell(3) = 5 partitions, {u,g}: 2, o and d alone -> 10 per block; singletons only: 1
    assert len(M.block_partitions(True)) == 10
    assert len(M.block_partitions(False)) == 1


def _instance(rng, B, nq, fused_discount=0.7):
    a = rng.uniform(0.2, 3.0, (B, 7))
    err = np.sort(rng.uniform(0.01, 0.4, nq))[::-1].copy()      # lower error ...
    base = np.sort(rng.uniform(1.0, 3.0, nq))                    # ... costs more
    size = {"q": 1.0, "k": 0.25, "v": 0.25, "o": 1.0, "u": 3.5, "g": 3.5, "d": 3.5}
    cost = np.empty((12, nq))
    for t, grp in enumerate(M.GROUPS):
        s = sum(size[l] for l in grp)
        launch = 0.8 * (fused_discount if len(grp) > 1 else 1.0)   # fusion saves launch overhead
        cost[t] = launch + s * base
    return a, err, cost


def test_loose_budget_closed_form():
    rng = np.random.default_rng(0)
    a, err, cost = _instance(rng, 2, 3)
    loss, c, asg = M.solve_bruteforce(a, err, cost, 1e9)
    assert math.isclose(loss, a.sum() * err.min(), rel_tol=1e-12)   # every layer at the best quantizer


def test_tight_budget_is_cheapest_assignment():
    rng = np.random.default_rng(1)
    a, err, cost = _instance(rng, 1, 2)
    cheapest = min(sum(cost[g].min() for g in part) for part in M.block_partitions(True))
    loss, c, _ = M.solve_bruteforce(a, err, cost, cheapest)
    assert math.isclose(c, cheapest, rel_tol=1e-12)
    assert M.solve_bruteforce(a, err, cost, cheapest * 0.999)[2] is None


def test_no_fusion_benefit_means_same_optimum():
    # when a fused group costs exactly the sum of its members, fusion cannot help
    rng = np.random.default_rng(2)
    a, err, cost = _instance(rng, 1, 2)
    for t, grp in enumerate(M.GROUPS):
        if len(grp) > 1:
            cost[t] = sum(cost[M.GROUPS.index((l,))] for l in grp)
    for C in (12.0, 16.0, 20.0):
        f = M.solve_bruteforce(a, err, cost, C, fusion=True)
        n = M.solve_bruteforce(a, err, cost, C, fusion=False)
        assert math.isclose(f[0], n[0], rel_tol=1e-12) or (math.isinf(f[0]) and math.isinf(n[0]))


@pytest.mark.parametrize("seed,B,nq,fusion", [(3, 1, 2, True), (4, 1, 3, True), (5, 2, 2, True), (6, 1, 3, False),
                                              (7, 2, 2, False)])
def test_library_solver_matches_bruteforce(seed, B, nq, fusion):
    rng = np.random.default_rng(seed)
    a, err, cost = _instance(rng, B, nq)
    lo = sum(min(sum(cost[g].min() for g in part) for part in M.block_partitions(fusion)) for _ in range(B))
    hi = B * sum(cost[M.GROUPS.index((l,))].max() for l in M.LAYERS)
    for C in np.linspace(lo, hi, 4):
        ref = M.solve_bruteforce(a, err, cost, C, fusion)
        loss, c, g, q = QL.plan_msq(a, err, cost, C, fusion)
        assert math.isclose(loss, ref[0], rel_tol=1e-9, abs_tol=1e-12)
        assert c <= C * (1 + 1e-12)
        # the returned assignment is valid and has the reported loss and cost
        tot_l, tot_c = 0.0, 0.0
        for b in range(B):
            seen = set()
            for l in range(7):
                t = int(g[b, l])
                assert M.LAYERS[l] in M.GROUPS[t]
                assert all(q[b, M.LAYERS.index(m)] == q[b, l] for m in M.GROUPS[t])
                tot_l += a[b, l] * err[q[b, l]]
                if t not in seen:
                    seen.add(t)
                    tot_c += cost[t, q[b, l]]
            if not fusion:
                assert all(len(M.GROUPS[int(t)]) == 1 for t in g[b])
        assert math.isclose(tot_l, loss, rel_tol=1e-9) and math.isclose(tot_c, c, rel_tol=1e-9)


def test_infeasible_budget_raises():
    rng = np.random.default_rng(8)
    a, err, cost = _instance(rng, 1, 2)
    with pytest.raises(QL.QPError, match="CONFIG_MISMATCH"):
        QL.plan_msq(a, err, cost, 0.1)
