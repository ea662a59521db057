"""Oracle pins for TCQ decoding and tail-biting Viterbi encoding
(PIN-4, PIN-5, PIN-6, PIN-8)."""
import itertools
import os

import numpy as np

from . import golden_values as G  # noqa: E402
import pytest

from oracle import codebooks as cb
from oracle import decode, encode


def test_all_zero_stream_decodes_to_lut0():
    # all-zero bits -> every window index 0 -> LUT[0] repeated T/V times
    lut = np.random.default_rng(0).standard_normal((1 << 16, 2))
    out = decode.tcq_decode_stream(np.zeros(4 * 128, dtype=np.int8), 4, 16, lut)
    assert out.shape == (128, 2)
    assert np.array_equal(out, np.repeat(lut[:1], 128, axis=0))


def test_wraparound_window():
    # s*T/V = 8, L = 4 -> step 3's window reads bits {6, 7, 0, 1}
    bits = np.array([1, 0, 0, 0, 0, 0, 1, 1], dtype=np.int8)     # b6=1, b7=1, b0=1, b1=0
    w = decode.tcq_windows(bits, s=2, L=4)
    assert w.shape == (4,)
    assert w[3] == 0b1110
    assert w[0] == 0b1000


def _brute_force(v, lut, s, L):
    """min over all 2^N streams of ||dq(r) - v||^2, using only the decoder."""
    n = v.shape[0]
    N = n * s
    best, best_r = np.inf, None
    for r in range(1 << N):
        bits = np.array([(r >> (N - 1 - i)) & 1 for i in range(N)], dtype=np.int8)
        e = float(((decode.tcq_decode_stream(bits, s, L, lut) - v) ** 2).sum())
        if e < best:
            best, best_r = e, bits
    return best, best_r


@pytest.mark.parametrize("L,V,s,T", [(4, 1, 2, 4), (6, 2, 2, 8), (8, 2, 3, 8)])
def test_exact_tailbiting_equals_brute_force(L, V, s, T):
    rng = np.random.default_rng(L * 100 + s)
    n = T // V
    for trial in range(4):
        lut = rng.standard_normal((1 << L, V))
        v = rng.standard_normal((1, n, V))
        bf, _ = _brute_force(v[0], lut, s, L)
        c, w = encode.tailbite_exact(v, lut, s, L)
        assert abs(c[0] - bf) < 1e-12
        bits = encode.windows_to_bits(w, s, L)[0]
        assert abs(((decode.tcq_decode_stream(bits, s, L, lut) - v[0]) ** 2).sum() - c[0]) < 1e-12
        c_rh, _ = encode.tailbite_rotate_half(v, lut, s, L)
        assert c_rh[0] >= bf - 1e-12              # every heuristic is >= the exact optimum


def test_fixed_start_viterbi_equals_brute_force_with_that_start():
    L, V, s, T = 6, 2, 2, 8
    n = T // V
    rng = np.random.default_rng(9)
    lut = rng.standard_normal((1 << L, V))
    v = rng.standard_normal((1, n, V))
    N = n * s
    for S in range(1 << (L - s)):
        best = np.inf
        for r in range(1 << N):
            bits = np.array([(r >> (N - 1 - i)) & 1 for i in range(N)], dtype=np.int8)
            w0 = decode.tcq_windows(bits, s, L)[0]
            if (w0 >> s) != S:
                continue
            best = min(best, float(((decode.tcq_decode_stream(bits, s, L, lut) - v[0]) ** 2).sum()))
        c, w = encode.viterbi_fixed(v, lut, s, L, np.array([S]))
        assert abs(c[0] - best) < 1e-12


def test_achievability_zero_error():
    # S (quant_engines): input equal to a decodable path's reconstruction -> error 0
    rng = np.random.default_rng(3)
    L, s = 8, 3
    lut = rng.standard_normal((1 << L, 2))
    bits = rng.integers(0, 2, 8 * s).astype(np.int8)
    v = decode.tcq_decode_stream(bits, s, L, lut)[None]
    c, w = encode.tailbite_rotate_half(v, lut, s, L)
    assert c[0] < 1e-24


def test_tailbiting_invariant_of_encoded_paths():
    # PIN-4: w_{n-1} mod 2^{L-s} == w_0 >> s, and decoding the stream returns the windows
    rng = np.random.default_rng(4)
    L, s = 10, 4
    lut = rng.standard_normal((1 << L, 2))
    v = rng.standard_normal((3, 128, 2))
    _, w = encode.tailbite_rotate_half(v, lut, s, L)
    assert np.all((w[:, -1] & ((1 << (L - s)) - 1)) == (w[:, 0] >> s))
    bits = encode.windows_to_bits(w, s, L)
    assert np.array_equal(decode.tcq_windows(bits, s, L), w)


def test_rotate_half_near_exact_at_T256():
    # reading R4: rotate-half reaches the exact tail-biting optimum in ~all T=256 trials (L=8)
    rng = np.random.default_rng(6)
    L, s = 8, 4
    lut = rng.standard_normal((1 << L, 2))
    v = rng.standard_normal((6, 128, 2))
    ce, _ = encode.tailbite_exact(v, lut, s, L)
    cr, _ = encode.tailbite_rotate_half(v, lut, s, L)
    assert np.all(cr >= ce - 1e-9)
    assert np.mean((cr - ce) / ce) < 2e-3


def _frozen_tlut(codebook_dir, tb):
    p = os.path.join(codebook_dir, f"tcq_tlut_tb{tb}.f16")
    if not os.path.exists(p):
        pytest.skip("codebooks not built")
    return np.fromfile(p, dtype="<f2").astype(np.float64).reshape(-1, 2)


# Table 5 TCQ-2 (within 2%) and the Fig. 2 ordering at every width: tests/test_oracle_scaling.py
# (with the rate-dependent reconstruction scale of reading R22).


def test_tcq2_L12_distortion(codebook_dir):
    # config C1 (L=12, reading R1): ~0.078, above the bound and above the L=16 figure
    lut = cb.quantlut_sym(_frozen_tlut(codebook_dir, 9), 12, 9)
    v = np.random.default_rng(77).standard_normal((32, 128, 2))
    c, _ = encode.tailbite_rotate_half(v, lut, 4, 12)
    d = c.sum() / v.size
    assert 0.0625 < d < 0.085


def test_distortion_decreases_with_rate(codebook_dir):
    lut = cb.quantlut_sym(_frozen_tlut(codebook_dir, 9), 12, 9)
    v = np.random.default_rng(8).standard_normal((16, 128, 2))
    ds = [encode.tailbite_rotate_half(v, lut, s, 12)[0].sum() / v.size for s in (3, 4, 5)]
    assert ds[0] > ds[1] > ds[2]
    for s, d in zip((3, 4, 5), ds):
        assert d >= 2.0 ** (-s)               # 2^(-2b), b = s/2
