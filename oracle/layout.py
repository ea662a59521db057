"""The frozen code layout (LAYOUT.md), implemented independently from the CUDA side.

TEST INFRASTRUCTURE (see oracle/__init__.py). Parity of this module is pinned only by
"oracle == GPU under the written contract" (the layout is ours, not the paper's);
its internal consistency is pinned by tests (bijection, exact storage size).

Summary of LAYOUT.md:
* Weights W[d_out][d_in] (nn.Linear orientation, reading R11) are cut into tiles of
  32 rows x 256 columns, stored row-tile-major: tile (rt, kt) follows (rt, kt-1).
* Inside a tile, lane l = 4g + q (g = l >> 2, q = l & 3) owns 128 consecutive "steps";
  step j = 8*kappa + 4*m + rho holds the weight pair
      row = 16*m + g + 8*(rho & 1),  cols = 64*q + 4*kappa + 2*(rho >> 1) + {0, 1}
  (a TCQ trellis of T = 256 weights = 4 rows x 64 columns, V = 2 pairs along d_in).
* Each step costs c bits (TCQ: c = s = 2b; VQ: c = 2b index bits, P:1004;
  NUQ/UNIF: c = 2b, the pair (even col, odd col) of b-bit codes, even code first).
  Lane l's stream is 128*c bits = 4c little-endian uint32 words, MSB-first
  (stream bit t = bit 31 - (t mod 32) of word t // 32). Word i of lane l sits at byte
      tile_base + ((i // 4) * 32 + l) * 16 + (i % 4) * 4.
  Tile bytes = 512 * c.
* Half-TCQ: k-tiles kt < KT/2 use s_lo = 2b, the rest s_hi = 2b + 1.
"""
from __future__ import annotations

import numpy as np

TILE_ROWS = 32
TILE_COLS = 256
LANES = 32
STEPS = 128


def step_position(lane: int, j: int) -> tuple[int, int]:
    """(row, first col) inside the 32 x 256 tile of step j of lane `lane`."""
    g, q = lane >> 2, lane & 3
    kappa, m, rho = j >> 3, (j >> 2) & 1, j & 3
    return 16 * m + g + 8 * (rho & 1), 64 * q + 4 * kappa + 2 * (rho >> 1)


def step_positions() -> np.ndarray:
    """[32 lanes][128 steps][2] -> (row, col) of the first weight of each pair."""
    out = np.zeros((LANES, STEPS, 2), dtype=np.int64)
    for lane in range(LANES):
        for j in range(STEPS):
            out[lane, j] = step_position(lane, j)
    return out


def scheme_step_bits(scheme: str, bits_x4: int) -> tuple[int, int]:
    """(c_lo, c_hi): bits per step for k-tiles in the first / second half of d_in."""
    if scheme == "tcq":
        assert bits_x4 % 2 == 0
        return bits_x4 // 2, bits_x4 // 2
    if scheme == "half_tcq":
        assert bits_x4 % 2 == 1
        s_lo = (bits_x4 - 1) // 2
        return s_lo, s_lo + 1
    if scheme == "vq":
        assert bits_x4 % 2 == 0
        return bits_x4 // 2, bits_x4 // 2
    if scheme in ("nuq", "unif"):
        assert bits_x4 % 4 == 0
        return bits_x4 // 2, bits_x4 // 2
    raise ValueError(scheme)


def tile_step_bits(scheme: str, bits_x4: int, kt: int, KT: int) -> int:
    c_lo, c_hi = scheme_step_bits(scheme, bits_x4)
    return c_lo if kt < KT // 2 else c_hi


def tile_offsets(d_out: int, d_in: int, scheme: str, bits_x4: int) -> tuple[np.ndarray, int]:
    """Byte offset of every tile [RT][KT] and the total code bytes."""
    RT, KT = d_out // TILE_ROWS, d_in // TILE_COLS
    offs = np.zeros((RT, KT), dtype=np.int64)
    pos = 0
    for rt in range(RT):
        for kt in range(KT):
            offs[rt, kt] = pos
            pos += 512 * tile_step_bits(scheme, bits_x4, kt, KT)
    return offs, pos


def lane_word_offsets(lane: int, nwords: int) -> np.ndarray:
    i = np.arange(nwords)
    return ((i // 4) * 32 + lane) * 16 + (i % 4) * 4


def read_lane_words(tile: np.ndarray, lane: int, c: int) -> np.ndarray:
    """The 4c uint32 stream words of `lane` from a tile's bytes (little-endian)."""
    offs = lane_word_offsets(lane, 4 * c)
    b = tile.astype(np.uint64)
    return (b[offs] | (b[offs + 1] << 8) | (b[offs + 2] << 16) | (b[offs + 3] << 24)).astype(np.uint64)


def words_to_bits(words: np.ndarray) -> np.ndarray:
    """MSB-first bit sequence of a word stream."""
    w = np.asarray(words, dtype=np.uint64)
    sh = np.arange(31, -1, -1, dtype=np.uint64)
    return ((w[:, None] >> sh[None, :]) & np.uint64(1)).astype(np.int64).reshape(-1)


def bits_to_words(bits: np.ndarray) -> np.ndarray:
    bits = np.asarray(bits, dtype=np.uint64).reshape(-1, 32)
    sh = np.arange(31, -1, -1, dtype=np.uint64)
    return np.bitwise_or.reduce(bits << sh[None, :], axis=1)


def write_lane_words(tile: np.ndarray, lane: int, words: np.ndarray) -> None:
    offs = lane_word_offsets(lane, len(words))
    w = np.asarray(words, dtype=np.uint64)
    for k in range(4):
        tile[offs + k] = ((w >> np.uint64(8 * k)) & np.uint64(0xFF)).astype(np.uint8)
