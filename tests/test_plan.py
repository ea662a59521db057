"""qp_optimal_bits (host-only C ABI, Theorem 1) against the oracle's allocation
(oracle/allocation.py, itself pinned by KKT / brute force in test_oracle_allocation.py).
The library is host code here: these tests run without a GPU."""
import numpy as np
import pytest

from oracle import allocation as A
from paper_2509_20214_b200 import _lib as QL


@pytest.mark.parametrize("seed", range(6))
def test_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    L = int(rng.integers(1, 40))
    a = rng.lognormal(0.0, 2.0, L)
    n = rng.integers(1, 64, L).astype(float) * 2 ** 16
    eta = float(rng.uniform(0.0, 2.5))
    M = float(rng.uniform(eta, eta + 4.0)) * n.sum()
    b = QL.optimal_bits(a, n, M, eta)
    ref = A.optimal_bits(a, n, M, eta)
    assert np.allclose(b, ref, atol=1e-9)
    assert abs((b * n).sum() - M) <= 1e-9 * M


def test_c5_allocation():
    shapes = [(4096, 4096), (1024, 4096), (1024, 4096), (4096, 4096), (14336, 4096), (14336, 4096), (4096, 14336)]
    n = np.array([o * i for o, i in shapes], dtype=float)
    b = QL.optimal_bits(np.ones(7), n, 3.25 * n.sum(), 1.5)
    assert np.round(b, 2).tolist() == [3.94, 4.94, 4.94, 3.94, 3.04, 3.04, 3.04]


def test_errors():
    n = np.ones(3)
    with pytest.raises(QL.QPError, match="CONFIG_MISMATCH"):
        QL.optimal_bits(np.ones(3), n, 1.0, 1.5)
    with pytest.raises(QL.QPError, match="INVALID_ARG"):
        QL.optimal_bits(np.array([1.0, -1.0, 1.0]), n, 10.0, 1.5)
