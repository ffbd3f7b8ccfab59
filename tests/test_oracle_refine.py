"""Pins for the oracle's NEXT-f1 refinement: TPS evaluation/gradient and the L-BFGS-B optimum."""
import numpy as np
import pytest


def test_tps_eval_reproduces_fit_and_gradient(O):
    rng = np.random.default_rng(0)
    x = rng.uniform(0, 1, size=(60, 2))
    y = np.sin(2 * x[:, 0]) * np.cos(3 * x[:, 1])
    fitted, w, beta = O.tps_fit(x, y, 1e-6)
    for i in range(0, 60, 7):
        assert O.tps_eval(x, w, beta, x[i])[0] == pytest.approx(fitted[i], abs=1e-10)
    p = np.array([0.37, 0.61])
    f0, g = O.tps_eval(x, w, beta, p)
    h = 1e-6
    for j in range(2):
        e = np.zeros(2); e[j] = h
        fd = (O.tps_eval(x, w, beta, p + e)[0] - O.tps_eval(x, w, beta, p - e)[0]) / (2 * h)
        assert g[j] == pytest.approx(fd, rel=1e-5, abs=1e-8)       # S:324 FD check


def test_refine_finds_known_maximum(O):
    # a smooth bump sampled on a 15 x 15 grid: the TPS optimum is within the interpolation error of
    # the analytic maximiser (0.31, 0.58)
    g = (np.arange(15) + 0.5) / 15
    x = np.array([[a, b] for a in g for b in g])
    y = 0.9 + 0.05 * np.exp(-((x[:, 0] - 0.31) ** 2 + (x[:, 1] - 0.58) ** 2) * 4)
    xs, fs, lam = O.refine(x, y, 0.0)
    assert np.allclose(xs, [0.31, 0.58], atol=3e-3)
    assert fs == pytest.approx(0.95, abs=2e-4)
    # maximum on the box boundary: a plane is maximised at the corner of the site box
    y2 = 1.0 + 0.1 * x[:, 0] - 0.2 * x[:, 1]
    xs2, fs2, _ = O.refine(x, y2, 0.0)
    assert np.allclose(xs2, [x[:, 0].max(), x[:, 1].min()], atol=1e-9)
