"""Pins of oracle/allocation.py (Theorem 1) against what the mathematics fixes:
KKT stationarity of the convex problem, closed-form special cases and brute force."""
import itertools
import math

import numpy as np
import pytest

from oracle import allocation as A

LN2 = math.log(2.0)


def test_uniform_when_layers_identical():
    # equal a_l and n_l: by symmetry and strict convexity the optimum is b = M / sum n
    n = np.full(5, 4096.0 * 4096.0)
    b = A.optimal_bits(np.ones(5), n, 3.25 * n.sum(), 1.5)
    assert np.allclose(b, 3.25, atol=1e-12)


def test_budget_is_tight_and_floor_respected():
    rng = np.random.default_rng(0)
    a = rng.uniform(0.1, 10.0, 12)
    n = rng.integers(1, 64, 12).astype(float) * 1024.0
    M = 3.0 * n.sum()
    b = A.optimal_bits(a, n, M, 1.5)
    assert abs((b * n).sum() - M) <= 1e-9 * M
    assert np.all(b >= 1.5 - 1e-12)


def test_kkt_conditions():
    # Lagrangian L = sum a 2^(-2b) + lam (sum b n - M) - sum mu (b - eta):
    # d/db_l: -2 ln2 a_l 2^(-2 b_l) + lam n_l - mu_l = 0, mu_l >= 0, mu_l (b_l - eta) = 0.
    # => g_l = 2 ln2 a_l 2^(-2 b_l) / n_l equals lam on free layers and is <= lam on clamped ones.
    rng = np.random.default_rng(1)
    a = rng.lognormal(0.0, 2.0, 20)
    n = rng.integers(1, 16, 20).astype(float) * 2 ** 20
    eta = 2.0
    b = A.optimal_bits(a, n, 3.0 * n.sum(), eta)
    g = 2 * LN2 * a * np.power(2.0, -2 * b) / n
    free = b > eta + 1e-9
    assert free.sum() >= 2 and (~free).sum() >= 1          # the case exercises both branches
    lam = g[free].mean()
    assert np.allclose(g[free], lam, rtol=1e-9)
    assert np.all(g[~free] <= lam * (1 + 1e-9))


def test_feasibility_edge_and_infeasible():
    n = np.array([1.0, 2.0, 3.0])
    b = A.optimal_bits(np.array([1.0, 5.0, 0.2]), n, 1.5 * n.sum(), 1.5)
    assert np.allclose(b, 1.5)
    with pytest.raises(ValueError):
        A.optimal_bits(np.ones(3), n, 1.4 * n.sum(), 1.5)


@pytest.mark.parametrize("a,n", [((1.0, 4.0), (1.0, 1.0)), ((3.0, 0.5, 1.0), (2.0, 1.0, 1.0)),
                                 ((1.0, 1.0, 1.0), (16.0, 4.0, 56.0))])
def test_brute_force_small(a, n):
    # exhaustive search over a 1/64-bit grid of every allocation that meets the budget
    a, n = np.array(a), np.array(n)
    eta, avg = 1.5, 3.0
    M = avg * n.sum()
    b = A.optimal_bits(a, n, M, eta)
    grid = np.arange(eta, 7.0 + 1e-9, 1 / 64)
    best = math.inf
    for combo in itertools.product(grid, repeat=len(a) - 1):
        rest = (M - float(np.dot(combo, n[:-1]))) / n[-1]       # last layer takes the rest of the budget
        if rest < eta:
            continue
        best = min(best, A.objective(a, list(combo) + [rest]))
    # the closed form is at least as good as every grid point, and within grid resolution of the best
    assert A.objective(a, b) <= best + 1e-12
    assert A.objective(a, b) >= best * (1 - 2e-3)


def test_llama_decoder_layer_c5():
    # Llama-3.1-8B decoder layer, a_l = 1, eta = 1.5, M = 3.25 b/weight avg.
    # With equal a_l, b_l - b_l' = ln(n_l'/n_l) / (2 ln 2): k/v (1024x4096) sit exactly 1 bit above
    # q/o (4096x4096), the MLP (14336x4096) log2(3.5)/2 below.
    shapes = [(4096, 4096), (1024, 4096), (1024, 4096), (4096, 4096), (14336, 4096), (14336, 4096), (4096, 14336)]
    n = np.array([o * i for o, i in shapes], dtype=float)
    b = A.optimal_bits(np.ones(7), n, 3.25 * n.sum(), 1.5)
    assert abs(b[1] - b[0] - 1.0) < 1e-9 and abs(b[2] - b[1]) < 1e-12
    assert abs(b[0] - b[4] - math.log2(3.5) / 2) < 1e-9
    assert np.round(b, 2).tolist() == [3.94, 4.94, 4.94, 3.94, 3.04, 3.04, 3.04]
