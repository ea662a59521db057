"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the Q-Palette method (no decoding, hashing,
rotation or matvec): only random-number generation with fixed seeds, following
the input recipe in DESIGN.md ("Input recipe") / SURVEY.md §8(d):

* weights for quality/parity: W ~ N(0, 1) iid, NumPy PCG64 seed 0;
* activations: x ~ N(0, 1) rounded to fp16, seed 1;
* per-output-channel scales: U(0.5, 1.5) / sqrt(d_in), fp32, seed 3;
* code streams for throughput: uniform random 32-bit words from splitmix64
  (seed 1000 + layer_id) -- every window / index then equally likely.

Both the oracle side and the CUDA side receive these arrays as *inputs*.
"""
from __future__ import annotations

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_words(seed: int, n_words32: int) -> np.ndarray:
    """n_words32 uniform uint32 words from the splitmix64 stream seeded with `seed`.

    Counter form: z_i = mix(seed + (i + 1) * gamma); each 64-bit output is split
    into (low, high) uint32 words. Vectorised, deterministic across platforms.
    """
    n64 = (n_words32 + 1) // 2
    with np.errstate(over="ignore"):
        i = np.arange(1, n64 + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z.view(np.uint32)[:n_words32].copy()


def random_code_bytes(n_bytes: int, layer_id: int = 0) -> np.ndarray:
    """Uniform random code bytes (throughput workload), seed 1000 + layer_id."""
    assert n_bytes % 4 == 0
    return splitmix64_words(1000 + layer_id, n_bytes // 4).view(np.uint8)


def gaussian_weights(d_out: int, d_in: int, seed: int = 0) -> np.ndarray:
    """W ~ N(0,1) iid, [d_out][d_in] float64 (PCG64)."""
    return np.random.Generator(np.random.PCG64(seed)).standard_normal((d_out, d_in))


def activations_fp16(batch: int, d_in: int, seed: int = 1) -> np.ndarray:
    """x ~ N(0,1) rounded to fp16, [batch][d_in]."""
    g = np.random.Generator(np.random.PCG64(seed))
    return g.standard_normal((batch, d_in)).astype(np.float16)


def channel_scales(d_out: int, d_in: int, seed: int = 3) -> np.ndarray:
    """Per-output-channel scales s_j ~ U(0.5, 1.5)/sqrt(d_in), fp32."""
    g = np.random.Generator(np.random.PCG64(seed))
    return (g.uniform(0.5, 1.5, size=d_out) / np.sqrt(d_in)).astype(np.float32)


def gaussian_vectors(n: int, dim: int, seed: int) -> np.ndarray:
    """n samples of a dim-dimensional standard Gaussian (codebook training data)."""
    return np.random.Generator(np.random.PCG64(seed)).standard_normal((n, dim))
