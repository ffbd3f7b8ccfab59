"""Pins for the oracle's thin-plate-spline smoother, GCV and argmax (Sec. 2.3)."""
import numpy as np
import pytest
from scipy.interpolate import RBFInterpolator


def _sites(N, d, seed=0):
    return np.random.default_rng(seed).uniform(0, 1, size=(N, d))


def test_interpolation_at_lambda_zero(O):
    x = _sites(60, 2)
    y = np.sin(3 * x[:, 0]) + x[:, 1] ** 2
    fitted, w, beta = O.tps_fit(x, y, 0.0)
    assert np.allclose(fitted, y, atol=1e-8)
    # side conditions T^T w = 0
    assert abs(w.sum()) < 1e-8 and np.allclose(x.T @ w, 0, atol=1e-8)


def test_affine_reproduced_for_any_lambda(O):
    x = _sites(50, 2, 1)
    y = 0.3 + 2 * x[:, 0] - 1.5 * x[:, 1]
    for lam in [0.0, 1e-6, 1e-2, 1.0]:
        fitted, w, beta = O.tps_fit(x, y, lam)
        assert np.allclose(fitted, y, atol=1e-9)
        assert np.allclose(w, 0, atol=1e-8)
        assert np.allclose(beta, [0.3, 2, -1.5], atol=1e-8)


@pytest.mark.parametrize("d,kernel", [(1, "cubic"), (2, "thin_plate_spline"), (3, "linear")])
def test_matches_scipy_rbf(O, d, kernel):
    # scipy's RBFInterpolator solves (K + s I) w + P b = y, P^T w = 0 with degree-1 P:
    # the same penalised TPS with s = N lambda (phi: d=1 r^3, d=2 r^2 log r, d=3 -r).
    x = _sites(80, d, 2)
    y = np.cos(2 * x.sum(1)) + 0.01 * np.random.default_rng(3).normal(size=80)
    for lam in [0.0, 1e-5, 1e-3]:
        fitted, _, _ = O.tps_fit(x, y, lam)
        ref = RBFInterpolator(x, y, kernel=kernel, smoothing=80 * lam, degree=1)(x)
        assert np.allclose(fitted, ref, atol=1e-8)


def test_gcv_influence_matrix_properties(O):
    x = _sites(40, 2, 4)
    A = O.tps_influence(x, 1e-3)
    assert np.allclose(A, A.T, atol=1e-9)                 # symmetric smoother
    ev = np.linalg.eigvalsh(A)
    assert ev.min() > -1e-9 and ev.max() < 1 + 1e-9      # shrinkage in [0, 1]
    assert np.sum(np.isclose(ev, 1, atol=1e-7)) >= 3     # affine space passes unchanged


def test_gcv_picks_smoothing_for_noisy_data(O):
    rng = np.random.default_rng(5)
    x = _sites(120, 2, 6)
    f = np.exp(-((x - 0.5) ** 2).sum(1) * 4)
    y = f + 0.05 * rng.normal(size=120)
    sm, lam = O.tps_smooth(x, y, -1.0)
    assert lam > 1e-10
    assert np.sqrt(np.mean((sm - f) ** 2)) < np.sqrt(np.mean((y - f) ** 2))
    # lam is the grid minimiser of the GCV score
    scores = [O.gcv_score(x, y, 10.0 ** g) for g in O.GCV_LOG10_GRID]
    assert lam == pytest.approx(10.0 ** O.GCV_LOG10_GRID[int(np.argmin(scores))])


def test_residual_sum_of_squares_monotone_in_lambda(O):
    x = _sites(50, 2, 7)
    y = np.random.default_rng(8).normal(size=50)
    rss = [np.sum((O.tps_fit(x, y, l)[0] - y) ** 2) for l in [0, 1e-6, 1e-4, 1e-2, 1]]
    assert all(a <= b + 1e-12 for a, b in zip(rss, rss[1:]))


def test_argmax_lowest_index_on_ties(O):
    assert O.argmax([0.1, 0.5, 0.5, 0.2]) == 1
    assert O.argmax([3.0]) == 0
    v = np.random.default_rng(9).normal(size=1000)
    assert O.argmax(v) == int(np.argmax(v))
