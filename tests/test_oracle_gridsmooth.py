"""Pins for the oracle's C4 dense-grid smoother (SURVEY §8(a) a9 "Dense regular grids (C4)";
DESIGN.md §2.13, reading R23): the separable Gaussian Nadaraya-Watson smoother and its GCV."""
import math

import numpy as np
import pytest


def _nw_2d_brute(P, xr, xa, hr, ha):
    # the 2-D Nadaraya-Watson estimate written as one double sum over all grid points with the
    # product Gaussian weight (no separable factorisation)
    nr, na = P.shape
    out = np.zeros_like(P)
    for i in range(nr):
        for j in range(na):
            num = den = 0.0
            for k in range(nr):
                for l in range(na):
                    w = math.exp(-0.5 * (((xr[i] - xr[k]) / hr) ** 2 + ((xa[j] - xa[l]) / ha) ** 2))
                    num += w * P[k, l]
                    den += w
            out[i, j] = num / den
    return out


def test_separable_equals_2d_double_sum(O):
    rng = np.random.default_rng(3)
    xr, xa = np.sort(rng.uniform(0, 1, 5)), np.sort(rng.uniform(0, 2, 7))
    P = rng.normal(size=(5, 7))
    for hr, ha in [(0.1, 0.3), (0.4, 0.05), (2.0, 1.0)]:
        got, _ = O.grid_kernel_smooth(P, xr, xa, hr, ha)
        assert np.allclose(got, _nw_2d_brute(P, xr, xa, hr, ha), rtol=0, atol=1e-13)


def test_constant_preserved_and_limits(O):
    xr, xa = np.linspace(0.05, 0.95, 12), np.linspace(0.001, 0.024, 9)
    P = np.full((12, 9), 0.937)
    for hr, ha in [(0.01, 0.0005), (0.2, 0.01), (10.0, 1.0)]:
        got, _ = O.grid_kernel_smooth(P, xr, xa, hr, ha)
        assert np.allclose(got, 0.937, rtol=0, atol=1e-15)
    rng = np.random.default_rng(5)
    Q = rng.normal(size=(12, 9))
    # h -> 0: the identity (tr S = n); h -> infinity: the global mean (tr S = 1)
    got, tr = O.grid_kernel_smooth(Q, xr, xa, 1e-4, 1e-6)
    assert np.allclose(got, Q, atol=1e-14) and tr == pytest.approx(108.0, abs=1e-9)
    got, tr = O.grid_kernel_smooth(Q, xr, xa, 1e6, 1e6)
    assert np.allclose(got, Q.mean(), atol=1e-9) and tr == pytest.approx(1.0, abs=1e-9)


def test_linear_reproduced_in_the_interior(O):
    # a symmetric kernel on a uniform grid reproduces linear functions exactly where the window is
    # complete (here >= 8 bandwidths from every edge: neglected weight exp(-32))
    xr, xa = np.linspace(0, 1, 81), np.linspace(0, 0.025, 61)
    P = 0.3 + 0.7 * xr[:, None] - 11.0 * xa[None, :]
    hr, ha = 1.0 * (xr[1] - xr[0]), 1.5 * (xa[1] - xa[0])
    got, _ = O.grid_kernel_smooth(P, xr, xa, hr, ha)
    ir = slice(9, 81 - 9)
    ia = slice(13, 61 - 13)
    assert np.allclose(got[ir, ia], P[ir, ia], rtol=0, atol=1e-12)
    # ...but not at the boundary (Nadaraya-Watson boundary bias)
    assert abs(got[0, 30] - P[0, 30]) > 1e-3


def test_trace_is_the_kronecker_operator_trace(O):
    rng = np.random.default_rng(8)
    xr, xa = np.sort(rng.uniform(0, 1, 6)), np.sort(rng.uniform(0, 1, 4))
    hr, ha = 0.2, 0.35
    P = rng.normal(size=(6, 4))
    Sr, Sa = O.kernel_matrix_nw(xr, hr), O.kernel_matrix_nw(xa, ha)
    K = np.kron(Sr, Sa)             # vec_row(S_r P S_a^T) = (S_r kron S_a) vec_row(P)
    got, tr = O.grid_kernel_smooth(P, xr, xa, hr, ha)
    assert np.allclose(K @ P.ravel(), got.ravel(), atol=1e-14)
    assert tr == pytest.approx(np.trace(K), rel=1e-14)
    res = P.ravel() - K @ P.ravel()
    n = P.size
    assert O.grid_gcv(P, xr, xa, hr, ha) == pytest.approx((res @ res / n) / (1 - np.trace(K) / n) ** 2, rel=1e-12)


def test_gcv_choice_tracks_the_noise(O):
    rng = np.random.default_rng(1)
    x, y = np.linspace(0, 1, 40), np.linspace(0, 1, 30)
    X, Y = np.meshgrid(x, y, indexing="ij")
    F = np.exp(-((X - 0.3) ** 2 + (Y - 0.6) ** 2) * 4)
    _, (hr, ha) = O.grid_smooth(F, x, y)
    assert hr == pytest.approx(0.5 * x[1]) and ha == pytest.approx(0.5 * y[1])    # noiseless: least smoothing
    _, (hr, ha) = O.grid_smooth(rng.normal(size=(40, 30)), x, y)
    assert hr >= 8 * x[1] and ha >= 8 * y[1]                                        # pure noise: heavy smoothing
    # the chosen pair is the grid minimiser
    P = F + 0.05 * rng.normal(size=F.shape)
    _, (hr, ha) = O.grid_smooth(P, x, y)
    g0 = O.grid_gcv(P, x, y, hr, ha)
    for kr in O.GRID_H_STEPS:
        for ka in O.GRID_H_STEPS:
            assert O.grid_gcv(P, x, y, kr * x[1], ka * y[1]) >= g0 - 1e-15
