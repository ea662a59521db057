"""The hot-path result y = diag(s) W_hat R x and the offline weight path (oracle, float64).

TEST INFRASTRUCTURE (see oracle/__init__.py).

The fused kernel reaches exactly (up to rounding order) the plain definition
    y[beta] = s (.) (W_hat @ (R x[beta]))
where W_hat = dq(codes) (oracle/decode.py), R the randomized Hadamard rotation
(oracle/rht.py) and s the per-output-channel scales. The oracle
computes it directly in float64.

Offline, data-free weight path (readings R10, R22):
    W' = W R^T (each row rotated), s_j = RMS(W'_j), W~ = W' / (s alpha), codes = encode(W~),
    stored scales s alpha (alpha = the codebook's rate-dependent reconstruction scale,
    oracle/scaling.py; 1 for NUQ / UNIF / VQ).
"""
from __future__ import annotations

import numpy as np

from . import decode, encode, rht


def linear_ref(W_hat: np.ndarray, scales: np.ndarray, x: np.ndarray, seed: int,
               prerotated: bool = False) -> np.ndarray:
    """y[batch][d_out] = s (.) (W_hat @ R x) in float64."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    xr = x if prerotated else rht.rht_apply(x, seed)
    return (xr @ np.asarray(W_hat, dtype=np.float64).T) * np.asarray(scales, dtype=np.float64)[None, :]


def linear_from_codes(codes, d_out, d_in, scheme, bits_x4, codebook, scales, x, seed, prerotated=False):
    W_hat = decode.decode_layer(codes, d_out, d_in, scheme, bits_x4, codebook)
    return linear_ref(W_hat, scales, x, seed, prerotated)


def gaussianize(W: np.ndarray, seed: int, alpha: float = 1.0) -> tuple[np.ndarray, np.ndarray]:
    """W' = W R^T, s_j = sqrt(mean_k W'_jk^2); returns (W' / (s alpha), s alpha) (readings
    R10, R22: the quantizer then sees unit-RMS rows shrunk by the reconstruction scale alpha)."""
    Wr = rht.rht_apply(np.asarray(W, dtype=np.float64), seed)     # row j -> R W_j
    s = np.sqrt(np.mean(Wr * Wr, axis=1)) * alpha
    return Wr / s[:, None], s


def quantize_offline(W: np.ndarray, scheme: str, bits_x4: int, codebook: dict, seed: int, alpha: float = 1.0):
    """Data-free quantization of one nn.Linear weight [d_out][d_in].
    Returns (codes uint8, scales float64 = s alpha)."""
    Wt, s = gaussianize(W, seed, alpha)
    return encode.encode_layer(Wt, scheme, bits_x4, codebook), s


def normwise_error(y: np.ndarray, y_ref: np.ndarray) -> np.ndarray:
    """Per batch row: max_j |y_j - y*_j| / max_j |y*_j| (reading R16)."""
    y = np.atleast_2d(np.asarray(y, dtype=np.float64))
    y_ref = np.atleast_2d(np.asarray(y_ref, dtype=np.float64))
    return np.max(np.abs(y - y_ref), axis=1) / np.max(np.abs(y_ref), axis=1)
