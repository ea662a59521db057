"""Oracle pins for the randomized Hadamard rotation (PIN-1, PIN-7)."""
import numpy as np
import pytest
import scipy.linalg

from oracle import rht


@pytest.mark.parametrize("b", [1, 2, 8, 64, 256])
def test_sylvester_orthogonality_exact(b):
    H = rht.sylvester(b)
    assert np.array_equal(H @ H.T, b * np.eye(b))          # integer-valued, exact


@pytest.mark.parametrize("b", [2, 16, 128])
def test_sylvester_matches_library(b):
    # scipy.linalg.hadamard is Sylvester's construction in natural order
    assert np.array_equal(rht.sylvester(b), scipy.linalg.hadamard(b).astype(float))


def test_h2_worked_example():
    # (1/sqrt 2) H_2 (1, 0)^T = (1/sqrt 2, 1/sqrt 2)^T with D = +I
    x = np.array([1.0, 0.0])
    y = rht.sylvester(2) @ x / np.sqrt(2)
    assert np.allclose(y, [2 ** -0.5, 2 ** -0.5], atol=0, rtol=1e-15)


def test_splitmix64_reference_vector():
    # splitmix64 with state 0: first output 0xE220A8397B1DCDAF, second 0x6E789E6AA1B965F4
    assert rht.splitmix64(0, 0) == 0xE220A8397B1DCDAF
    assert rht.splitmix64(0, 1) == 0x6E789E6AA1B965F4


def test_signs_balanced_and_deterministic():
    d = rht.rht_signs(7, 4096)
    assert set(np.unique(d)) == {-1.0, 1.0}
    assert abs(d.mean()) < 0.06
    assert np.array_equal(d, rht.rht_signs(7, 4096))


@pytest.mark.parametrize("d_in,b", [(256, 256), (4096, 4096), (14336, 2048), (28672, 4096), (8192, 8192), (768, 256)])
def test_block_size(d_in, b):
    assert rht.rht_block(d_in) == b


def test_rotation_is_orthogonal():
    R = rht.rht_matrix(512, seed=7, block=256)
    assert np.allclose(R @ R.T, np.eye(512), atol=1e-13)
    R2 = rht.rht_matrix(768, seed=3)          # 3 blocks of 256
    assert np.allclose(R2.T @ R2, np.eye(768), atol=1e-13)


def test_norm_preserved_and_inverse():
    x = np.random.default_rng(0).standard_normal((3, 14336))
    xr = rht.rht_apply(x, seed=7)
    assert np.allclose(np.linalg.norm(xr, axis=1), np.linalg.norm(x, axis=1), rtol=1e-12)


def test_unit_vector_closed_form():
    # PIN-7: x = e_0 -> x' = (d_0 / sqrt(b)) * 1 on block 0, zero elsewhere
    n, b = 1024, 256
    x = np.zeros((1, n)); x[0, 0] = 1.0
    xr = rht.rht_apply(x, seed=11, block=b)[0]
    d0 = rht.rht_signs(11, 1)[0]
    assert np.allclose(xr[:b], d0 / np.sqrt(b), rtol=1e-14)
    assert np.all(xr[b:] == 0)


def test_rotation_gaussianizes_spike():
    # a spiky row becomes flat (incoherence processing)
    x = np.zeros((1, 4096)); x[0, 17] = 100.0
    xr = rht.rht_apply(x, seed=1)[0]
    assert np.allclose(np.abs(xr), 100.0 / 64.0)
