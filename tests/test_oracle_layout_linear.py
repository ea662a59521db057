"""Oracle pins for the layout contract, storage size, RTN and the matvec
(PIN-2, PIN-7, PIN-10 definition)."""
import numpy as np
import pytest

from oracle import codebooks as cb
from oracle import decode, encode, layout, linear, rht


def test_step_map_is_a_bijection():
    pos = layout.step_positions()
    cover = np.zeros((32, 256), dtype=int)
    for lane in range(32):
        for j in range(128):
            r, c = pos[lane, j]
            cover[r, c] += 1
            cover[r, c + 1] += 1
    assert np.all(cover == 1)


def test_trellis_is_4_rows_by_64_cols():
    pos = layout.step_positions()
    for lane in range(32):
        rows = set(pos[lane, :, 0]); cols = set(pos[lane, :, 1])
        g, q = lane >> 2, lane & 3
        assert rows == {g, g + 8, g + 16, g + 24}
        assert cols == set(range(64 * q, 64 * q + 64, 2))


def test_step_map_matches_mma_fragment_order():
    # step j = 8*kappa + 4*m + rho is register rho of the m16n8k16 A fragment of (kappa, m):
    # rho&1 -> +8 rows, rho>>1 -> the second k-slot pair of the thread
    for lane in range(32):
        for kappa in range(16):
            for m in range(2):
                base = layout.step_position(lane, 8 * kappa + 4 * m)
                assert layout.step_position(lane, 8 * kappa + 4 * m + 1) == (base[0] + 8, base[1])
                assert layout.step_position(lane, 8 * kappa + 4 * m + 2) == (base[0], base[1] + 2)
                assert layout.step_position(lane, 8 * kappa + 4 * m + 3) == (base[0] + 8, base[1] + 2)


@pytest.mark.parametrize("scheme,bits_x4,d_out,d_in,expect", [
    ("tcq", 8, 4096, 4096, 4096 * 4096 * 2 // 8),
    ("tcq", 10, 14336, 4096, 14336 * 4096 * 5 // 16),
    ("half_tcq", 13, 4096, 4096, 6815744),                  # 4096*2048*3/8 + 4096*2048*3.5/8
    ("vq", 6, 256, 512, 256 * 512 * 3 // 16),               # VQ-1.5: 3 bits per pair
    ("nuq", 8, 256, 256, 256 * 256 * 2 // 8),               # 2-bit NUQ -> bits/8 bytes
    ("unif", 16, 64, 256, 64 * 256 * 4 // 8),
])
def test_storage_is_exactly_b_bits_per_weight(scheme, bits_x4, d_out, d_in, expect):
    _, total = layout.tile_offsets(d_out, d_in, scheme, bits_x4)
    assert total == expect
    assert total * 8 == d_out * d_in * bits_x4 // 4


def test_word_bit_roundtrip():
    bits = np.random.default_rng(0).integers(0, 2, 32 * 20)
    w = layout.bits_to_words(bits)
    assert np.array_equal(layout.words_to_bits(w), bits)
    assert layout.bits_to_words(np.r_[1, np.zeros(31, int)])[0] == 0x80000000     # MSB-first
    tile = np.zeros(512 * 5, dtype=np.uint8)
    for lane in range(32):
        layout.write_lane_words(tile, lane, w + lane)
    for lane in range(32):
        assert np.array_equal(layout.read_lane_words(tile, lane, 5), (w + lane).astype(np.uint64))


def test_decode_places_single_code():
    # one VQ-2 index at (tile (1, 1), lane 13, step 37) lands at its mapped position
    d_out, d_in, c = 64, 512, 4
    offs, total = layout.tile_offsets(d_out, d_in, "vq", 8)
    codes = np.zeros(total, dtype=np.uint8)
    lane, j, idx = 13, 37, 0b1011
    bits = np.zeros(128 * c, dtype=np.int64)
    bits[j * c:(j + 1) * c] = [1, 0, 1, 1]
    layout.write_lane_words(codes[offs[1, 1]:offs[1, 1] + 512 * c], lane, layout.bits_to_words(bits))
    lut2d = np.arange(32, dtype=float).reshape(16, 2) + 100
    W = decode.decode_layer(codes, d_out, d_in, "vq", 8, {"lut2d": lut2d})
    r, col = layout.step_position(lane, j)
    assert W[32 + r, 256 + col] == lut2d[idx, 0] and W[32 + r, 256 + col + 1] == lut2d[idx, 1]
    expect = np.tile(lut2d[0], (d_out, d_in // 2))            # all other codes are index 0
    expect[32 + r, 256 + col:256 + col + 2] = lut2d[idx]
    assert np.array_equal(W, expect)


def test_rtn_ties_lowest_index():
    # equidistant -> lower index; exact codeword -> zero error
    lut = np.array([-1.0, 0.0, 1.0, 3.0])
    assert encode.nuq_rtn(np.array([0.5, -0.5, 2.0, 1.0]), lut).tolist() == [1, 0, 2, 2]
    lut1 = np.array([-0.79788, 0.79788])
    i = encode.nuq_rtn(np.array([0.1]), lut1)[0]
    assert i == 1 and abs((0.1 - lut1[i]) ** 2 - 0.4870) < 1e-4


@pytest.mark.parametrize("scheme,bits_x4", [("nuq", 8), ("nuq", 12), ("vq", 8), ("unif", 8)])
def test_encode_decode_roundtrip_on_codewords(scheme, bits_x4):
    # a matrix made of codewords reconstructs exactly (S quantize_matrix example)
    rng = np.random.default_rng(1)
    d_out, d_in = 64, 512
    if scheme == "vq":
        lut2d = rng.standard_normal((1 << (bits_x4 // 2), 2))
        idx = rng.integers(0, len(lut2d), (d_out, d_in // 2))
        W = lut2d[idx].reshape(d_out, d_in)
        book = {"lut2d": lut2d}
    else:
        lut = np.sort(rng.standard_normal(1 << (bits_x4 // 4)))
        W = lut[rng.integers(0, len(lut), (d_out, d_in))]
        book = {"lut": lut}
    codes = encode.encode_layer(W, scheme, bits_x4, book)
    assert np.array_equal(decode.decode_layer(codes, d_out, d_in, scheme, bits_x4, book), W)


def test_half_tcq_codes_split_along_d_in():
    # W[:, :d_in/2] at b, W[:, d_in/2:] at b+0.5 -> tile widths s_lo, s_hi
    assert layout.scheme_step_bits("half_tcq", 11) == (5, 6)        # 2.75 = 2.5 | 3.0
    offs, total = layout.tile_offsets(32, 512, "half_tcq", 11)
    assert offs[0, 1] == 512 * 5 and total == 512 * 11


def test_matvec_closed_forms():
    # PIN-7: x = e_0 -> y_j = s_j d_0 / sqrt(b) * sum_{k<b} W_hat[j, k]
    rng = np.random.default_rng(2)
    d_out, d_in = 32, 512
    Wh = rng.standard_normal((d_out, d_in)); s = rng.uniform(0.5, 1.5, d_out)
    x = np.zeros((1, d_in)); x[0, 0] = 1.0
    y = linear.linear_ref(Wh, s, x, seed=5)
    d0 = rht.rht_signs(5, 1)[0]
    assert np.allclose(y[0], s * d0 / np.sqrt(512) * Wh[:, :512].sum(1), rtol=1e-12)
    # constant weights c -> y_j = s_j c sum_k x'_k
    xr = rht.rht_apply(rng.standard_normal((2, d_in)), 5)
    y2 = linear.linear_ref(np.full((d_out, d_in), 0.25), s, xr, seed=5, prerotated=True)
    assert np.allclose(y2, 0.25 * s[None] * xr.sum(1)[:, None], rtol=1e-12)


def test_gaussianize_is_exact_without_quantization():
    # y = (W R^T)(R x): rotation + per-channel scaling is lossless before quantization
    rng = np.random.default_rng(3)
    W = rng.standard_normal((64, 768)) * rng.uniform(0.1, 3, (64, 1))
    x = rng.standard_normal((3, 768))
    Wt, s = linear.gaussianize(W, seed=9)
    assert np.allclose(np.sqrt(np.mean(Wt ** 2, axis=1)), 1.0, rtol=1e-12)
    assert np.allclose(linear.linear_ref(Wt, s, x, seed=9), x @ W.T, rtol=1e-10, atol=1e-12)


def test_normwise_error_definition():
    y_ref = np.array([[1.0, -4.0, 0.0]]); y = np.array([[1.1, -4.0, 0.2]])
    assert np.allclose(linear.normwise_error(y, y_ref), [0.05])


def test_c1_end_to_end_quantize(codebook_dir):
    # config C1: 256x256 TCQ-2.0, L=12, tlut_bits 9, W ~ N(0,1) seed 0
    import os
    p = os.path.join(codebook_dir, "tcq_tlut_tb9.f16")
    if not os.path.exists(p):
        pytest.skip("codebooks not built")
    from qp_synth import gaussian_weights
    tl = np.fromfile(p, dtype="<f2").astype(np.float64).reshape(-1, 2)
    book = {"lut": cb.quantlut_sym(tl, 12, 9), "L": 12}
    W = gaussian_weights(256, 256, seed=0)
    codes, s = linear.quantize_offline(W, "tcq", 8, book, seed=7)
    assert codes.size == 256 * 256 * 2 // 8
    Wt, s2 = linear.gaussianize(W, seed=7)
    Wh = decode.decode_layer(codes, 256, 256, "tcq", 8, book)
    dist = np.mean((Wh - Wt) ** 2) / np.mean(Wt ** 2)
    assert 0.0625 < dist < 0.085                              # >= 2^(-2b), ~0.078 (reading R1)
    x = np.random.default_rng(1).standard_normal((1, 256))
    y = linear.linear_ref(Wh, s, x, seed=7)
    y_true = x @ W.T
    assert np.linalg.norm(y - y_true) / np.linalg.norm(y_true) < 0.35
