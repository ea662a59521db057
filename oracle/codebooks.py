"""Codebooks of the Q-Palette quantizers (oracle side, float64).

TEST INFRASTRUCTURE (see oracle/__init__.py). Every codebook used by the GPU
path is produced by `scripts/build_codebooks.py`, which calls only this module,
and is frozen to fp16 (RNE) once; both sides then load the same fp16 bytes
(reading R7: the frozen fp16 values are normative).

Paper passages (P:n = /root/reference/PAPER.md line n):
  NUQ   P:977-982  "flash1dkmeans ... 10^8 randomly sampled standard Gaussian values ... k=2^b"
  VQ    P:997-1001 "scikit-learn ... Lloyd's algorithm ... max_iter=300 and tol=1e-6 ... k=2^{2b}"
  TCQ   P:1022-1036 tlut by k-means of 2^20 2-D Gaussian samples "with appropriate scaling",
        expanded by the verbatim `quantlut_sym` listing; L=16, tlut_bits 9 (b<=4), 10 (4.5), 11 (5.0)
  Unif  P:251 ("Unif" baseline of Fig. 2; grid unspecified -> reading R15)
"""
from __future__ import annotations

import numpy as np
from scipy import optimize, stats

# --------------------------------------------------------------------------------------
# NUQ: Lloyd-Max scalar quantizer of N(0,1)
# --------------------------------------------------------------------------------------


def _cell_moments(a: np.ndarray, b: np.ndarray):
    """P(a<X<b), E[X 1{a<X<b}], E[X^2 1{a<X<b}] for X ~ N(0,1) (exact)."""
    Pa, Pb = stats.norm.cdf(a), stats.norm.cdf(b)
    fa, fb = stats.norm.pdf(a), stats.norm.pdf(b)
    with np.errstate(invalid="ignore"):
        afa = np.where(np.isinf(a), 0.0, a * fa)
        bfb = np.where(np.isinf(b), 0.0, b * fb)
    p0 = Pb - Pa
    p1 = fa - fb
    p2 = p0 - (bfb - afa)
    return p0, p1, p2


def scalar_mse(levels: np.ndarray) -> float:
    """Exact E[(X - Q(X))^2], X ~ N(0,1), Q = nearest level (thresholds at midpoints)."""
    c = np.sort(np.asarray(levels, dtype=np.float64))
    t = np.concatenate([[-np.inf], (c[:-1] + c[1:]) / 2, [np.inf]])
    p0, p1, p2 = _cell_moments(t[:-1], t[1:])
    return float(np.sum(p2 - 2 * c * p1 + c * c * p0))


def nuq_lloyd_max(bits: int, tol: float = 1e-14, max_iter: int = 200000) -> np.ndarray:
    """2^bits Lloyd-Max levels for N(0,1): the population limit of the paper's 1-D
    k-means on 10^8 Gaussian samples. Fixed point of
      t_i = (c_i + c_{i+1}) / 2,   c_i = E[X | t_{i-1} < X < t_i].
    Pinned: NUQ-2 distortion 0.11747, NUQ-1 = 1 - 2/pi (closed form)."""
    k = 1 << bits
    c = stats.norm.ppf((np.arange(k) + 0.5) / k)
    for _ in range(max_iter):
        t = np.concatenate([[-np.inf], (c[:-1] + c[1:]) / 2, [np.inf]])
        p0, p1, _ = _cell_moments(t[:-1], t[1:])
        c_new = p1 / p0
        if np.max(np.abs(c_new - c)) < tol:
            c = c_new
            break
        c = c_new
    return c


def unif_levels(bits: int, delta: float) -> np.ndarray:
    """Symmetric uniform grid (i - (2^b - 1)/2) * delta, i = 0..2^b-1 (reading R15)."""
    k = 1 << bits
    return (np.arange(k) - (k - 1) / 2.0) * delta


def unif_optimal(bits: int) -> tuple[np.ndarray, float]:
    """MSE-optimal uniform grid for N(0,1) (Max 1960): returns (levels, delta).
    Pinned by the textbook values delta = 0.9957 / 0.5860 / 0.3352 (b = 2/3/4)."""
    res = optimize.minimize_scalar(lambda d: scalar_mse(unif_levels(bits, d)),
                                   bounds=(1e-3, 4.0), method="bounded",
                                   options={"xatol": 1e-12})
    return unif_levels(bits, res.x), float(res.x)


# --------------------------------------------------------------------------------------
# k-means (scikit-learn Lloyd, as the paper states for VQ and the TCQ tlut)
# --------------------------------------------------------------------------------------


def kmeans_2d(samples: np.ndarray, k: int, seed: int, max_iter: int = 300, tol: float = 1e-6) -> np.ndarray:
    """scikit-learn Lloyd k-means (max_iter=300, tol=1e-6); returns k x 2 centroids."""
    from sklearn.cluster import KMeans
    km = KMeans(n_clusters=k, init="k-means++", n_init=1, max_iter=max_iter, tol=tol,
                random_state=seed, algorithm="lloyd")
    km.fit(samples)
    return np.asarray(km.cluster_centers_, dtype=np.float64)


def vq_codebook(bits: float, samples: np.ndarray, seed: int, max_iter: int = 300) -> np.ndarray:
    """2-D VQ LUT in R^{2^{2b} x 2}. Sorted lexicographically for determinism
    (entry order is arbitrary; codes index whatever order is frozen). Absolute centroid
    values: parity unpinned (pinned only statistically through Table 5)."""
    k = int(round(2 * bits))
    cb = kmeans_2d(samples, 1 << k, seed, max_iter=max_iter)
    order = np.lexsort((cb[:, 1], cb[:, 0]))
    return cb[order]


def tcq_tlut(tlut_bits: int, samples: np.ndarray, seed: int, max_iter: int = 300) -> np.ndarray:
    """tlut in R^{2^tlut_bits x 2}: k-means of 2-D Gaussian samples, then
    "appropriate scaling" read as unit second moment per coordinate under uniform index
    sampling (reading R6; pinned by TCQ-2 distortion 0.07101)."""
    cb = kmeans_2d(samples, 1 << tlut_bits, seed, max_iter=max_iter)
    order = np.lexsort((cb[:, 1], cb[:, 0]))
    cb = cb[order]
    return cb / np.sqrt(np.mean(cb * cb))


def tlut_bits_for(bits: float) -> int:
    """tlut_bits = 9 for b <= 4, 10 for 4.5, 11 for 5.0."""
    if bits <= 4.0:
        return 9
    if bits <= 4.5:
        return 10
    return 11


# --------------------------------------------------------------------------------------
# quantlut_sym, verbatim, with the constants generalised for L != 16
# --------------------------------------------------------------------------------------


def quantlut_sym(tlut: np.ndarray, L: int, tlut_bits: int) -> np.ndarray:
    """Hybrid codebook LUT in R^{2^L x 2}. For L = 16 this is the paper's listing line by line:
        lut = arange(1 << L); lut = (lut + 1) * lut
        sflp = 1 - ((lut >> 15) & 1) * 2
        lut = (lut >> (16 - tlut_bits - 1)) & ((1 << tlut_bits) - 1)
        lut = tlut[lut]; lut[:, 0] = lut[:, 0] * sflp
    For L != 16 (config C1 uses L = 12, reading R1) the constants 15 and 16 become L-1 and L
    and the product is taken mod 2^L."""
    lut = np.arange(1 << L, dtype=np.int64)
    lut = ((lut + 1) * lut) % (1 << L)
    sflp = 1 - ((lut >> (L - 1)) & 1) * 2
    lut = (lut >> (L - tlut_bits - 1)) & ((1 << tlut_bits) - 1)
    out = np.array(tlut, dtype=np.float64)[lut]
    out[:, 0] = out[:, 0] * sflp
    return out


def freeze_fp16(a: np.ndarray) -> np.ndarray:
    """Round once to fp16 (RNE); the fp16 values are normative (reading R7)."""
    return np.asarray(a, dtype=np.float64).astype(np.float16)
