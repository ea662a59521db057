"""Rate-dependent "appropriate scaling" of the TCQ codebook (oracle side, float64).

TEST INFRASTRUCTURE (see oracle/__init__.py).

P:1022-1023: the tlut is obtained by k-means on 2-D Gaussian samples "with appropriate scaling".
The frozen tlut files keep the unit second moment of reading R6 (one table per tlut_bits,
shared by every width that uses it, so decode is unchanged and bit-exact); the scaling itself is
a per-(width, tlut_bits, L) factor alpha applied on the weight side (reading R22):

    encode   W~ = W' / (s * alpha)          (the standardized weights seen by the trellis)
    decode   W_hat = dq(codes),  stored scale s * alpha,  y = diag(s * alpha) W_hat R x

so the per-weight reconstruction is alpha * dq(r). alpha_b minimises the Gaussian distortion
(Table 5's metric)

    D_b(alpha) = E || v - alpha * dq(RTN(v / alpha)) ||^2 / T,   v ~ N(0, I_T)

which is what the paper's scaling must achieve for P:298 ("TCQ-based schemes ... consistently
achieve quantization error close to theoretical lower bounds, outperforming simpler
quantizers") to hold at every rate: one fixed scale cannot be right at 2 bits (where the
trellis' reachable set is sparse and the codewords should shrink toward the mode) and at 4.5 bits
(where the codewords should spread to the Gaussian's support). Pinned by: the Fig. 2 ordering
TCQ < VQ < NUQ at every width, TCQ-2 within 2% of Table 5, D_b >= 2^(-2b), and
local optimality of each frozen alpha (tests/test_oracle_scaling.py).

Half-TCQ stores one scale per row, so its two halves share one alpha: the
minimiser of the mean of the two halves' distortions (each with the shared LUT, reading R12).
"""
from __future__ import annotations

import numpy as np

from . import encode


def tcq_distortion(v: np.ndarray, lut: np.ndarray, s: int, L: int, alpha: float) -> float:
    """D(alpha) on trellis vectors v [nb][T/2][2]: encode v/alpha with the rotate-half tail-biting
    Viterbi (reading R4) and measure || v - alpha * dq ||^2 per weight. The Viterbi path cost of
    v/alpha is sum || v/alpha - dq ||^2, so the distortion is alpha^2 * cost / (nb * T)."""
    v = np.asarray(v, dtype=np.float64)
    cost, _ = encode.tailbite_rotate_half(v / alpha, lut, s, L)
    return float(alpha * alpha * cost.sum() / v.size)


def golden_min(f, a: float, b: float, tol: float = 2e-3):
    """Golden-section minimisation of a unimodal f on [a, b]; returns (x, f(x), evaluations)."""
    g = (np.sqrt(5.0) - 1.0) / 2.0
    c, d = b - g * (b - a), a + g * (b - a)
    fc, fd = f(c), f(d)
    ev = [(c, fc), (d, fd)]
    while b - a > tol:
        if fc <= fd:
            b, d, fd = d, c, fc
            c = b - g * (b - a)
            fc = f(c)
            ev.append((c, fc))
        else:
            a, c, fc = c, d, fd
            d = a + g * (b - a)
            fd = f(d)
            ev.append((d, fd))
    x, fx = min(ev, key=lambda t: t[1])
    return x, fx, ev
