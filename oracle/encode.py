"""Quantization (encoding) of the palette quantizers (oracle side, float64).

TEST INFRASTRUCTURE (see oracle/__init__.py).

  NUQ RTN  argmin_r |v - LUT[int(r)]|
  VQ  RTN  argmin_r ||v - LUT[int(r)]||_2
  TCQ RTN  "the Viterbi algorithm to find the optimal binary representation r in
           {0,1}^{sT/V} that is dequantized into the vector closest to v",
           with tail-biting windows.
  Ties go to the lowest index (RTN) / lowest predecessor (Viterbi) (reading R5).

Trellis notation: window w_i (L bits) dequantizes step i; the state after step i is
sigma_i = w_i mod 2^{L-s}; the next window is w_{i+1} = k * 2^{L-s} + sigma' with
w_{i+1} >> s = sigma_i. The stream r is the concatenation of the top s bits of each
window; tail-biting requires sigma_{n-1} = w_0 >> s (the state "before" step 0).

Three encoders:
  viterbi_fixed     exact DP for a fixed start state S (= required end state)
  tailbite_exact    min over all S of viterbi_fixed (reading R4: the exact tail-biting optimum)
  tailbite_rotate_half  normative for real sizes (reading R4): roll v by T/2, free-start
                    Viterbi, read the state at the original wrap boundary, fixed-S pass.
"""
from __future__ import annotations

import numpy as np

INF = np.inf


def nuq_rtn(v: np.ndarray, lut: np.ndarray) -> np.ndarray:
    """Nearest-entry index for scalars (first index on ties)."""
    v = np.asarray(v, dtype=np.float64)
    d = np.abs(v[..., None] - np.asarray(lut, dtype=np.float64))
    return np.argmin(d, axis=-1)


def vq_rtn(v: np.ndarray, lut2d: np.ndarray) -> np.ndarray:
    """Nearest-entry index for 2-D vectors v[..., 2] (first index on ties)."""
    v = np.asarray(v, dtype=np.float64)
    lut2d = np.asarray(lut2d, dtype=np.float64)
    d = ((v[..., None, :] - lut2d) ** 2).sum(-1)
    return np.argmin(d, axis=-1)


def _step_costs(v_i: np.ndarray, lut: np.ndarray) -> np.ndarray:
    """||v_i - LUT[w]||^2 for all windows w: [nb][2^L]."""
    return ((v_i[:, None, :] - lut[None, :, :]) ** 2).sum(-1)


def viterbi(v: np.ndarray, lut: np.ndarray, s: int, L: int, start: np.ndarray | None,
            end: np.ndarray | None):
    """Batched Viterbi over nb sequences.

    v: [nb][n][V]; lut: [2^L][V]; start: [nb] start states (w_0 >> s) or None = free;
    end: [nb] required end states sigma_{n-1} or None = free (argmin, lowest index).
    Returns (cost [nb], windows [nb][n])."""
    v = np.asarray(v, dtype=np.float64)
    lut = np.asarray(lut, dtype=np.float64)
    nb, n, _ = v.shape
    ns = 1 << (L - s)
    D = np.zeros((nb, ns))
    if start is not None:
        D[:] = INF
        D[np.arange(nb), start] = 0.0
    w_all = np.arange(1 << L)
    prev = w_all >> s
    bp = np.empty((n, nb, ns), dtype=np.int32)
    for i in range(n):
        E = D[:, prev] + _step_costs(v[:, i, :], lut)          # [nb][2^L]
        E = E.reshape(nb, 1 << s, ns)                           # w = k * 2^{L-s} + sigma'
        k = np.argmin(E, axis=1)                                # lowest k on ties
        D = np.take_along_axis(E, k[:, None, :], axis=1)[:, 0, :]
        bp[i] = k
    if end is None:
        sig = np.argmin(D, axis=1)
    else:
        sig = np.asarray(end)
    cost = D[np.arange(nb), sig]
    windows = np.empty((nb, n), dtype=np.int64)
    for i in range(n - 1, -1, -1):
        k = bp[i, np.arange(nb), sig]
        w = k * ns + sig
        windows[:, i] = w
        sig = w >> s
    return cost, windows


def windows_to_bits(windows: np.ndarray, s: int, L: int) -> np.ndarray:
    """Stream r = concat_i (top s bits of w_i), MSB-first: [nb][n*s]."""
    top = windows >> (L - s)
    sh = np.arange(s - 1, -1, -1)
    bits = (top[..., None] >> sh) & 1
    return bits.reshape(windows.shape[0], -1).astype(np.int8)


def viterbi_fixed(v, lut, s, L, S):
    """Exact optimum among tail-biting paths whose start state (w_0 >> s) and end state are S."""
    S = np.asarray(S)
    return viterbi(v, lut, s, L, S, S)


def tailbite_exact(v, lut, s, L):
    """Exact tail-biting optimum: min over all 2^{L-s} start states (tiny configs only)."""
    v = np.asarray(v, dtype=np.float64)
    nb = v.shape[0]
    best_c = np.full(nb, INF)
    best_w = np.zeros((nb, v.shape[1]), dtype=np.int64)
    for S in range(1 << (L - s)):
        c, w = viterbi_fixed(v, lut, s, L, np.full(nb, S))
        better = c < best_c
        best_c[better] = c[better]
        best_w[better] = w[better]
    return best_c, best_w


def tailbite_rotate_half(v, lut, s, L):
    """Rotate-half tail-biting encoder (reading R4, normative):
    1. roll v by T/2 (n/2 steps); 2. free-start Viterbi, argmin end state;
    3. trace back to the state at the original wrap boundary (after rolled step n - n/2 - 1);
    4. fixed-S Viterbi on the unrolled v with that S."""
    v = np.asarray(v, dtype=np.float64)
    nb, n, _ = v.shape
    h = n // 2
    rolled = np.concatenate([v[:, h:], v[:, :h]], axis=1)
    _, w_r = viterbi(rolled, lut, s, L, None, None)
    S = w_r[:, n - h - 1] & ((1 << (L - s)) - 1)
    return viterbi_fixed(v, lut, s, L, S)


# --------------------------------------------------------------------------------------
# Whole-layer data-free encoding into the LAYOUT.md tile format
# --------------------------------------------------------------------------------------


def encode_layer(Wt: np.ndarray, scheme: str, bits_x4: int, codebook: dict, chunk: int = 64) -> np.ndarray:
    """Codes (uint8, LAYOUT.md order) of a standardized matrix Wt[d_out][d_in].

    Data-free procedure: partition into scalars (NUQ), pairs (VQ) or T-vectors (TCQ),
    RTN each independently, concatenate. TCQ uses tailbite_rotate_half."""
    from . import layout
    d_out, d_in = Wt.shape
    RT, KT = d_out // 32, d_in // 256
    offs, total = layout.tile_offsets(d_out, d_in, scheme, bits_x4)
    codes = np.zeros(total, dtype=np.uint8)
    pos = layout.step_positions()
    # gather every (tile, lane) vector of 128 pairs
    for half in (0, 1):
        kts = [kt for kt in range(KT) if (kt >= KT // 2) == bool(half)]
        if not kts:
            continue
        c = layout.tile_step_bits(scheme, bits_x4, kts[0], KT)
        tiles = [(rt, kt) for rt in range(RT) for kt in kts]
        vecs = np.empty((len(tiles), 32, 128, 2))
        for ti, (rt, kt) in enumerate(tiles):
            rows = rt * 32 + pos[:, :, 0]
            cols = kt * 256 + pos[:, :, 1]
            vecs[ti, :, :, 0] = Wt[rows, cols]
            vecs[ti, :, :, 1] = Wt[rows, cols + 1]
        flat = vecs.reshape(-1, 128, 2)
        if scheme in ("tcq", "half_tcq"):
            L = codebook["L"]
            bits = np.empty((flat.shape[0], 128 * c), dtype=np.int8)
            for b0 in range(0, flat.shape[0], chunk):
                _, w = tailbite_rotate_half(flat[b0:b0 + chunk], codebook["lut"], c, L)
                bits[b0:b0 + chunk] = windows_to_bits(w, c, L)
        else:
            if scheme == "vq":
                idx = vq_rtn(flat, codebook["lut2d"])
            else:
                bsc = c // 2
                lut = codebook["lut"]
                idx = (nuq_rtn(flat[..., 0], lut) << bsc) | nuq_rtn(flat[..., 1], lut)
            sh = np.arange(c - 1, -1, -1)
            bits = ((idx[..., None] >> sh) & 1).reshape(flat.shape[0], -1).astype(np.int8)
        bits = bits.reshape(len(tiles), 32, -1)
        for ti, (rt, kt) in enumerate(tiles):
            tile = codes[offs[rt, kt]: offs[rt, kt] + 512 * c]
            for lane in range(32):
                layout.write_lane_words(tile, lane, layout.bits_to_words(bits[ti, lane]))
    return codes
