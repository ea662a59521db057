"""Randomized Hadamard rotation of the activations (oracle side, float64).

TEST INFRASTRUCTURE (see oracle/__init__.py).

Paper: "rotating weights only along the input dimension (W -> RW) and applying
per-output-channel scaling ... reduces the number of online rotations per
Transformer block from 14 to 4" (§3.3). The online side rotates the
activations, x' = R x, so that y = (W R^T)(R x).

Readings:
  R8  R = (1/sqrt(b)) * blockdiag(H_b, ..., H_b) * D, H_b Sylvester (natural order),
      H_b[i][j] = (-1)^popcount(i & j); D = diag(d_0..d_{n-1}),
      d_i = -1 if bit 63 of splitmix64(seed, i) is set else +1.
  R9  b = largest power-of-two divisor of d_in (d_in = 14336 = 7 * 2^11 -> b = 2048).

This is an explicit matrix product with Sylvester entries (no butterfly), so it is
independent of the GPU fast Walsh-Hadamard transform.
"""
from __future__ import annotations

import numpy as np

_MASK = (1 << 64) - 1


def splitmix64(seed: int, i: int) -> int:
    """i-th output (i >= 0) of the splitmix64 counter generator: mix(seed + (i+1)*gamma)."""
    z = (seed + (i + 1) * 0x9E3779B97F4A7C15) & _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


def rht_signs(seed: int, n: int) -> np.ndarray:
    """d_i in {+1, -1} for i < n (reading R8), one splitmix64 call per index."""
    return np.array([-1.0 if (splitmix64(seed, i) >> 63) & 1 else 1.0 for i in range(n)])


def rht_block(d_in: int) -> int:
    """Largest power-of-two divisor of d_in (reading R9)."""
    if d_in <= 0:
        raise ValueError("d_in must be positive")
    return d_in & (-d_in)


def sylvester_rows(rows: np.ndarray, b: int) -> np.ndarray:
    """Rows `rows` of the b x b Sylvester Hadamard matrix, entries (-1)^popcount(i & j)."""
    j = np.arange(b, dtype=np.int64)
    par = np.bitwise_count(np.bitwise_and(rows[:, None].astype(np.int64), j[None, :])) & 1
    return 1.0 - 2.0 * par


def sylvester(b: int) -> np.ndarray:
    return sylvester_rows(np.arange(b), b)


def rht_apply(x: np.ndarray, seed: int, block: int | None = None) -> np.ndarray:
    """x' = R x for each row of x ([batch][d_in] -> [batch][d_in], float64).

    x'[beta, o*b + i] = (1/sqrt(b)) * sum_j H_b[i][j] * d_{o*b+j} * x[beta, o*b + j]."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    n = x.shape[1]
    b = rht_block(n) if block is None else block
    if n % b:
        raise ValueError("block must divide d_in")
    d = rht_signs(seed, n)
    xd = x * d[None, :]
    out = np.empty_like(xd)
    chunk = 512
    for o in range(n // b):
        seg = xd[:, o * b:(o + 1) * b]
        for r0 in range(0, b, chunk):
            rows = np.arange(r0, min(b, r0 + chunk))
            H = sylvester_rows(rows, b)
            out[:, o * b + r0:o * b + r0 + len(rows)] = seg @ H.T
    return out / np.sqrt(b)


def rht_matrix(n: int, seed: int, block: int | None = None) -> np.ndarray:
    """R as an explicit n x n matrix (small n only)."""
    return rht_apply(np.eye(n), seed, block).T
