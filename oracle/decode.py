"""Dequantization dq(r; LUT) of every palette quantizer (oracle side, float64).

TEST INFRASTRUCTURE (see oracle/__init__.py).

Definitions followed (P:n = /root/reference/PAPER.md line n):
  NUQ   dq(r; LUT) = LUT[int(r)],  r in {0,1}^b
  VQ    dq(r; LUT) = LUT[int(r)] in R^2, r in {0,1}^{2b}
  TCQ   dq(r; LUT) = concat_{i=0}^{T/V-1} LUT[r[i*s : i*s + L]], indices wrapping
        around the end of r (tail-biting), s = 2b, V = 2, L = 16, T = 256
  Half-TCQ  first half of d_in at b, second half at b + 0.5, one LUT
  UNIF  NUQ decode with a uniform LUT (reading R15)
Bit order of int(r): first stream bit is the most significant (reading R2).
Placement of the decoded values follows oracle/layout.py (LAYOUT.md).
"""
from __future__ import annotations

import numpy as np

from . import layout


def bits_to_int(bits: np.ndarray) -> np.ndarray:
    """int(r) of the last axis, first bit most significant."""
    n = bits.shape[-1]
    w = (1 << np.arange(n - 1, -1, -1)).astype(np.int64)
    return bits.astype(np.int64) @ w


def tcq_windows(bits: np.ndarray, s: int, L: int) -> np.ndarray:
    """Tail-biting windows int(r[i*s : i*s+L]) (indices mod len(r)) of bit streams [..., N]."""
    N = bits.shape[-1]
    n = N // s
    idx = (np.arange(n)[:, None] * s + np.arange(L)[None, :]) % N
    return bits_to_int(bits[..., idx])


def tcq_decode_stream(bits: np.ndarray, s: int, L: int, lut: np.ndarray) -> np.ndarray:
    """dq(r; LUT) for one TCQ bitstream r of length s*T/V: returns [T/V][2]."""
    return np.asarray(lut, dtype=np.float64)[tcq_windows(np.asarray(bits), s, L)]


def _tile_lane_bits(codes: np.ndarray, offs: np.ndarray, c: int) -> np.ndarray:
    """[ntiles][32][128*c] stream bits of the tiles starting at byte offsets `offs`."""
    nw = 4 * c
    lane_offs = np.stack([layout.lane_word_offsets(l, nw) for l in range(32)])  # [32][nw]
    byte_idx = offs[:, None, None] + lane_offs[None, :, :]                          # [t][32][nw]
    b = codes.astype(np.uint64)
    words = (b[byte_idx] | (b[byte_idx + 1] << 8) | (b[byte_idx + 2] << 16) | (b[byte_idx + 3] << 24))
    sh = np.arange(31, -1, -1, dtype=np.uint64)
    bits = (words[..., None] >> sh) & np.uint64(1)
    return bits.reshape(len(offs), 32, nw * 32).astype(np.int8)


def decode_layer(codes: np.ndarray, d_out: int, d_in: int, scheme: str, bits_x4: int,
                 codebook: dict, tile_chunk: int = 512) -> np.ndarray:
    """W_hat[d_out][d_in] (float64) from packed codes in LAYOUT.md order.

    codebook: {"lut": 2^L x 2, "L": L} for tcq / half_tcq (the full hybrid LUT of
    quantlut_sym), {"lut2d": 2^{2b} x 2} for vq, {"lut": 2^b} for nuq / unif."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    RT, KT = d_out // layout.TILE_ROWS, d_in // layout.TILE_COLS
    offs, total = layout.tile_offsets(d_out, d_in, scheme, bits_x4)
    if codes.size < total:
        raise ValueError(f"need {total} code bytes, got {codes.size}")
    pos = layout.step_positions()                      # [32][128][2]
    W = np.empty((d_out, d_in), dtype=np.float64)
    # group tiles by their bits-per-step (half-TCQ has two widths)
    for half in (0, 1):
        kts = [kt for kt in range(KT) if (kt >= KT // 2) == bool(half)]
        if not kts:
            continue
        c = layout.tile_step_bits(scheme, bits_x4, kts[0], KT)
        tiles = [(rt, kt) for rt in range(RT) for kt in kts]
        for t0 in range(0, len(tiles), tile_chunk):
            chunk = tiles[t0:t0 + tile_chunk]
            toffs = np.array([offs[rt, kt] for rt, kt in chunk], dtype=np.int64)
            bits = _tile_lane_bits(codes, toffs, c)     # [t][32][128c]
            if scheme in ("tcq", "half_tcq"):
                vals = np.asarray(codebook["lut"], dtype=np.float64)[tcq_windows(bits, c, codebook["L"])]
            else:
                idx = bits_to_int(bits.reshape(len(chunk), 32, 128, c))          # [t][32][128]
                if scheme == "vq":
                    vals = np.asarray(codebook["lut2d"], dtype=np.float64)[idx]
                else:
                    bsc = c // 2
                    lut = np.asarray(codebook["lut"], dtype=np.float64)
                    vals = np.stack([lut[idx >> bsc], lut[idx & ((1 << bsc) - 1)]], axis=-1)
            for ti, (rt, kt) in enumerate(chunk):
                rows = rt * 32 + pos[:, :, 0]
                cols = kt * 256 + pos[:, :, 1]
                W[rows, cols] = vals[ti, :, :, 0]
                W[rows, cols + 1] = vals[ti, :, :, 1]
    return W
