"""Optimal fractional bit allocation with ideal Gaussian quantizers (oracle, float64).

TEST INFRASTRUCTURE (see oracle/__init__.py).

Problem (Eq. mpq_frac): minimise  sum_l a_l 2^(-2 b_l)
                                   subject to sum_l b_l n_l <= M,  b_l >= eta,
with n_l = d_in_l * d_out_l. Theorem 1 gives the closed form

    b_l* = max{ eta, (1 / (2 ln 2)) ln(a_l / n_l) + C },

with the constant C that makes the budget tight, sum_l b_l* n_l = M (feasible iff
M >= eta sum_l n_l). The oracle follows the theorem step by step: the left-hand side
S(C) = sum_l max{eta, u_l + C} n_l is continuous and non-decreasing in C, so C is found
by bisection to float64 resolution; nothing else is approximated.

Pins (tests/test_oracle_allocation.py): the KKT conditions of the convex problem
(equal marginal a_l 2 ln2 2^(-2 b_l) / n_l on every layer above eta, larger on the
clamped ones), equal sensitivities and sizes -> the uniform allocation M / sum n,
the feasibility edge M = eta sum n -> all eta, and brute force over a fine grid on
2- and 3-layer problems.
"""
from __future__ import annotations

import math

import numpy as np


def optimal_bits(a, n, M: float, eta: float) -> np.ndarray:
    """Theorem 1: b_l* for sensitivities a_l > 0, sizes n_l > 0 (weights), total
    budget M (bits) and floor eta. Raises ValueError when M < eta * sum(n) (infeasible)."""
    a = np.asarray(a, dtype=np.float64)
    n = np.asarray(n, dtype=np.float64)
    if a.shape != n.shape or a.ndim != 1 or a.size == 0:
        raise ValueError("a and n must be non-empty 1-D arrays of equal length")
    if np.any(a <= 0) or np.any(n <= 0):
        raise ValueError("sensitivities and sizes must be positive")
    total = float(n.sum())
    if M < eta * total * (1 - 1e-12):
        raise ValueError("infeasible budget: M < eta * sum(n)")
    u = np.log(a / n) / (2.0 * math.log(2.0))        # (1 / (2 ln 2)) ln(a_l / n_l)

    def S(C):
        return float((np.maximum(eta, u + C) * n).sum())

    # bracket: at C_lo every layer sits at eta (S = eta * sum n <= M); at C_hi, S >= M
    lo = eta - float(u.max())
    hi = M / total - float(u.min())
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if S(mid) < M:
            lo = mid
        else:
            hi = mid
        if hi - lo <= 1e-15 * max(1.0, abs(hi)):
            break
    C = 0.5 * (lo + hi)
    return np.maximum(eta, u + C)


def objective(a, b) -> float:
    """sum_l a_l 2^(-2 b_l): the surrogate of Eq. mpq_frac."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float((a * np.power(2.0, -2.0 * b)).sum())
