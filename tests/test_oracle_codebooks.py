"""Oracle pins for the codebooks (PIN-3, PIN-6)."""
import hashlib
import json
import os

import numpy as np

from . import golden_values as G  # noqa: E402
import pytest

from oracle import codebooks as cb


def test_nuq1_closed_form():
    # S:140 / textbook: 2-level Lloyd-Max for N(0,1) is +-sqrt(2/pi), MSE 1 - 2/pi
    c = cb.nuq_lloyd_max(1)
    assert np.allclose(c, [-np.sqrt(2 / np.pi), np.sqrt(2 / np.pi)], rtol=1e-12)
    assert abs(cb.scalar_mse(c) - (1 - 2 / np.pi)) < 1e-12


def test_nuq2_matches_table5():
    # Ours-NUQ-2 mean distortion 0.11747 (std 4.24e-5); Lloyd-Max population optimum 0.117482
    mse = cb.scalar_mse(cb.nuq_lloyd_max(2))
    assert abs(mse - G.table5("nuq-2.0")) < 2e-4
    # textbook Max (1960) 4-level levels +-0.4528, +-1.5104
    assert np.allclose(cb.nuq_lloyd_max(2), [-1.5104, -0.4528, 0.4528, 1.5104], atol=1e-4)


@pytest.mark.parametrize("b,mse", [(3, 0.03455), (4, 0.009501)])
def test_nuq_textbook_mse(b, mse):
    assert abs(cb.scalar_mse(cb.nuq_lloyd_max(b)) - mse) < 2e-5


@pytest.mark.parametrize("b,delta,mse", [(2, 0.9957, 0.1188), (3, 0.5860, 0.03744), (4, 0.3352, 0.01154)])
def test_uniform_textbook(b, delta, mse):
    # Max (1960) optimum uniform quantizer for N(0,1)
    lv, d = cb.unif_optimal(b)
    assert abs(d - delta) < 1e-4
    assert abs(cb.scalar_mse(lv) - mse) < 1e-4


def test_scalar_mse_matches_monte_carlo():
    # the exact-integral MSE formula vs a sample mean (independent computation)
    x = np.random.default_rng(5).standard_normal(2_000_000)
    for c in (cb.nuq_lloyd_max(2), cb.unif_optimal(3)[0]):
        q = c[np.argmin(np.abs(x[:, None] - c[None, :]), axis=1)]
        assert abs(np.mean((x - q) ** 2) - cb.scalar_mse(c)) < 4e-4


def test_rate_distortion_bound_scalar():
    # E[err] >= 2^(-2b)
    for b in (1, 2, 3, 4, 5):
        assert cb.scalar_mse(cb.nuq_lloyd_max(b)) >= 2.0 ** (-2 * b)


def _hash_trace(i, L=16, tb=9):
    p = (i + 1) * i                       # full-width product, as in the listing
    sign = -1 if (p >> (L - 1)) & 1 else 1
    idx = (p >> (L - tb - 1)) & ((1 << tb) - 1)
    return p, sign, idx


def test_quantlut_sym_traces():
    # i=0 -> tlut[0]; i=181 -> p=32942, sign -1, idx 2
    tlut = np.random.default_rng(0).standard_normal((512, 2))
    lut = cb.quantlut_sym(tlut, 16, 9)
    assert lut.shape == (65536, 2)
    assert np.array_equal(lut[0], tlut[0])
    for case in G.load("quantlut_sym_trace.json")["cases"]:
        w = case["window"]
        p, sign, idx = _hash_trace(w)
        assert (p, sign, idx) == (case["p"], case["sign"], case["idx"])
        assert np.array_equal(lut[w], [case["sign"] * tlut[case["idx"], 0], tlut[case["idx"], 1]])
    for i in np.random.default_rng(1).integers(0, 65536, 200):
        p, sign, idx = _hash_trace(int(i))
        assert np.array_equal(lut[i], [sign * tlut[idx, 0], tlut[idx, 1]])


@pytest.mark.parametrize("L,tb,per_key", [(16, 9, 64), (16, 10, 32), (16, 11, 16), (12, 9, 4)])
def test_quantlut_key_uniformity(L, tb, per_key):
    # every (sign, idx) key is hit equally often over all 2^L windows (survey App. A)
    w = np.arange(1 << L, dtype=np.int64)
    p = ((w + 1) * w) % (1 << L)
    key = ((p >> (L - 1)) & 1) * (1 << tb) + ((p >> (L - tb - 1)) & ((1 << tb) - 1))
    counts = np.bincount(key, minlength=1 << (tb + 1))
    assert np.all(counts == per_key)


def test_quantlut_symmetry():
    # w and 2^L - 1 - w hash to the same entry: (w+1)w = (-w)(-w-1)
    tlut = np.random.default_rng(2).standard_normal((512, 2))
    lut = cb.quantlut_sym(tlut, 16, 9)
    assert np.array_equal(lut, lut[::-1])


def test_tlut_bits_rule():
    # P:1036
    assert [cb.tlut_bits_for(b) for b in (1.5, 2.0, 3.5, 4.0, 4.5, 5.0)] == [9, 9, 9, 9, 10, 11]


# ---- frozen codebook files -------------------------------------------------------------

def _manifest(codebook_dir):
    p = os.path.join(codebook_dir, "MANIFEST.json")
    if not os.path.exists(p):
        pytest.skip("codebooks not built")
    return json.load(open(p))


def _load(codebook_dir, name):
    return np.fromfile(os.path.join(codebook_dir, name + ".f16"), dtype="<f2")


def test_manifest_hashes(codebook_dir):
    man = _manifest(codebook_dir)
    for name, meta in man.items():
        data = open(os.path.join(codebook_dir, meta["file"]), "rb").read()
        assert hashlib.sha256(data).hexdigest() == meta["sha256"], name


def test_frozen_nuq_is_lloyd_max(codebook_dir):
    man = _manifest(codebook_dir)
    for b in (2, 3, 4):
        if f"nuq_b{b}" not in man:
            continue
        lv = _load(codebook_dir, f"nuq_b{b}").astype(np.float64)
        assert np.array_equal(lv, cb.nuq_lloyd_max(b).astype(np.float16).astype(np.float64))


def test_frozen_tlut_unit_second_moment(codebook_dir):
    man = _manifest(codebook_dir)
    for tb in (9, 10, 11):
        if f"tcq_tlut_tb{tb}" not in man:
            continue
        t = _load(codebook_dir, f"tcq_tlut_tb{tb}").astype(np.float64).reshape(-1, 2)
        assert t.shape[0] == 1 << tb
        assert abs(np.mean(t * t) - 1.0) < 2e-3


def test_frozen_vq2_matches_table5(codebook_dir):
    # Ours-VQ-2 mean distortion 0.10857 (k-means codebook, nearest-entry RTN)
    man = _manifest(codebook_dir)
    if "vq_c4" not in man:
        pytest.skip("vq_c4 not built")
    v = _load(codebook_dir, "vq_c4").astype(np.float64).reshape(-1, 2)
    assert v.shape == (16, 2)
    x = np.random.default_rng(123).standard_normal((1_000_000, 2))
    d = ((x[:, None, :] - v[None]) ** 2).sum(-1).min(1).mean() / 2
    ref = G.table5("vq-2.0")
    assert abs(d - ref) / ref < 0.02        # sklearn Lloyd on 2^20 samples: 0.1075 (-1.0%)
    assert d >= 2.0 ** -4                                   # P:162 bound
    assert d < cb.scalar_mse(cb.nuq_lloyd_max(2))           # Fig. 2 ordering NUQ > VQ
