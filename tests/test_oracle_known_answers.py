"""Known-answer cases of the reference's estimator tests, on the oracle
(pins the restatement independently of the golden runs)."""

import math

import numpy as np

from oracle import oracle


def test_idl_documented_weight_value():
    # N_y=4, sigma2=10, squared distance 80 -> raw weight exp(-1) (test_estimators.py:90-96)
    y0 = np.zeros(4)
    yj = np.full((1, 4), math.sqrt(20.0))
    vals, raw = oracle.idl(y0, np.zeros((1, 4)), yj, 10.0)
    assert abs(raw - math.exp(-1.0)) < 1e-12


def test_idl_three_candidate_oracle():
    y0 = np.array([10.0, 20.0, 30.0])
    x = np.array([[1, 2, 3, 4], [5, 6, 7, 8], [9, 10, 11, 12]], dtype=float)
    y = np.array([[10, 20, 31], [12, 20, 30], [10, 25, 30]], dtype=float)
    raws = [math.exp(-((yy - y0) ** 2).sum() / (2 * 10.0 * 3)) for yy in y]
    expected = sum(r * xx for r, xx in zip(raws, x)) / sum(raws)
    vals, raw = oracle.idl(y0, x, y, 10.0)
    assert np.allclose(vals, expected, atol=1e-12)
    assert abs(raw - sum(raws)) <= 1e-12 * sum(raws)


def test_idl_underflow():
    vals, raw = oracle.idl(np.zeros(2), np.ones((1, 4)), np.array([[1e8, 0.0]]), 10.0)
    assert vals is None and raw == 0.0


def test_brl_two_point_mean():
    assert oracle.brl(np.array([0.0, 255.0])).tolist() == [127.5] * 4


def straight_line_hql(y0, x, y):
    """Independent FP64 restatement with explicit inverses (cf. test_estimators.py:423-470)."""
    m, n = y.shape
    z = np.hstack([x, y])
    c = (z - z.mean(0)).T @ (z - z.mean(0)) / (m - 1)
    cxy, cyy = c[:4, 4:], c[4:, 4:]
    tr = np.trace(cyy)
    cyy = cyy + (1e-6 * tr / n if tr > 0 else 1e-6) * np.eye(n)
    inv = np.linalg.inv(cyy)

    def weights(center, beta, exclude=None):
        e = np.array([-((center - y[j]) @ inv @ (center - y[j])) / (2 * beta) if j != exclude else -np.inf
                      for j in range(m)])
        w = np.exp(e - e[np.isfinite(e)].max())
        if exclude is not None:
            w[exclude] = 0.0
        return w / w.sum()

    best, best_eps = None, np.inf
    for k in range(-8, 13):
        w = weights(y0, 2.0**k)
        eps = ((y0 - w @ y) ** 2).sum()
        if eps < best_eps:
            best_eps, best = eps, 2.0**k
    w = weights(y0, best)
    xt, yt = w @ x, w @ y
    order = np.argsort(((y - y0) ** 2).sum(1), kind="stable")[: min(n + 1, m)]
    num = den = 0.0
    for i in order:
        wi = weights(y[i], best, exclude=i)
        ci = cxy @ (inv @ (y[i] - wi @ y))
        num += (x[i] - wi @ x) @ ci
        den += ci @ ci
    alpha = 0.0 if den < 1e-12 else float(np.clip(num / den, 0, 4))
    return xt + alpha * (cxy @ (inv @ (y0 - yt))), best, alpha


def test_hql_matches_straight_line():
    rng = np.random.default_rng(21)
    for _ in range(8):
        m, n = int(rng.integers(4, 40)), int(rng.integers(2, 12))
        y0 = rng.uniform(0, 50, n)
        y = rng.uniform(0, 50, (m, n))
        x = rng.uniform(0, 50, (m, 4))
        vals, info = oracle.hql(y0, x, y)
        exp_vals, beta, alpha = straight_line_hql(y0, x, y)
        assert info["layer"] == 2
        assert info["beta"] == beta
        assert abs(info["alpha"] - alpha) < 1e-9
        assert np.allclose(vals, exp_vals, atol=1e-9)


def test_hql_ladder():
    vals, info = oracle.hql(np.array([10.0, 20.0]), np.zeros((0, 4)), np.zeros((0, 2)))
    assert info["layer"] == 0 and info["fallback"] and np.allclose(vals, 15.0)
    vals, info = oracle.hql(np.array([10.0, 20.0]), np.array([[1.0, 2, 3, 4]]), np.array([[10.0, 20.0]]))
    assert info["layer"] == 1 and info["fallback"] and np.allclose(vals, [1, 2, 3, 4])


def test_hql_identical_prototypes():
    rng = np.random.default_rng(19)
    v = np.array([4.0, 5.0, 6.0, 7.0])
    vals, info = oracle.hql(rng.uniform(0, 30, 3), np.tile(v, (6, 1)), rng.uniform(0, 30, (6, 3)))
    assert info["layer"] == 2 and info["alpha"] == 0.0
    assert np.allclose(vals, v, atol=1e-9)


def test_pairwise_sum_order_matches_numpy():
    # d2 in NumPy's pairwise order: BRL mean of 33 values is bit-identical to numpy
    rng = np.random.default_rng(0)
    for n in (1, 5, 8, 9, 16, 31, 32):
        y0 = rng.uniform(0, 255, n) * np.exp(rng.uniform(-5, 5, n))
        assert oracle.brl(y0)[0] == float(y0.mean())
