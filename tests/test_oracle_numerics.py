"""CPU: the oracle's restatement of NumPy's pairwise summation
(numpy/_core/src/umath/loops_utils.h.src, pairwise_sum) is bit-exact
against ndarray.sum on the lengths the path sums: context sizes (<= 32),
the alpha sums over 4k <= 132 elements (one split beyond 128) and longer
runs, on values with heavy cancellation."""

import numpy as np
import pytest

from oracle import oracle


@pytest.mark.parametrize("n", [0, 1, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 64, 127, 128, 129, 132, 200, 256, 257, 1000, 1849])
def test_pairwise_sum_bit_exact(n):
    rng = np.random.default_rng(1234 + n)
    for scale in (1.0, 1e8):
        a = rng.standard_normal(n) * scale + rng.standard_normal(n) * 1e-8
        assert oracle.pairwise_sum(a).hex() == float(a.sum()).hex(), (n, scale)


def test_pairwise_sum_is_not_sequential():
    # a case where the pairwise and the sequential orders differ: the oracle
    # must follow NumPy, not a left-to-right loop
    a = np.array([1e16] + [1.0] * 15 + [-1e16] + [1.0] * 15, dtype=np.float64)
    seq = 0.0
    for v in a:
        seq += v
    assert oracle.pairwise_sum(a) == a.sum()
    assert a.sum() != seq
