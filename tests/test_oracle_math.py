"""Pins for the oracle's normal CDF/quantile, Cholesky, Formula-1 correlation and MVN orthant."""
import math

import numpy as np
import pytest
from scipy import integrate, special, stats


def test_phi_inv_matches_library(O):
    ps = np.concatenate([np.logspace(-300, -1, 120), np.linspace(0.01, 0.99, 97), 1 - np.logspace(-16, -2, 30)])
    for p in ps:
        ref = special.ndtri(p)
        if ref == 0:
            continue
        assert abs(O.Phi_inv(p) - ref) <= 2e-15 * abs(ref) + 1e-300
    assert O.Phi_inv(0.5) == 0.0
    assert O.Phi_inv(0.975) == pytest.approx(1.959963984540054, abs=1e-15)


def test_phi_matches_library(O):
    for x in np.linspace(-37, 8, 200):
        assert O.Phi(x) == pytest.approx(special.ndtr(x), rel=1e-12, abs=1e-300)


def test_threshold_sentinel(O):
    assert math.isinf(O.threshold(0.0)) and O.threshold(0.0) > 0
    assert O.threshold(0.025) == pytest.approx(1.959963984540054, abs=1e-15)


def test_null_corr_formula1(O):
    S = O.null_corr([1, 0.5, 0.25])
    assert S[0, 1] == pytest.approx(0.707107, abs=1e-6)
    assert S[0, 2] == pytest.approx(0.5, abs=1e-15)
    assert S[1, 2] == pytest.approx(0.707107, abs=1e-6)
    assert np.allclose(S, S.T) and np.allclose(np.diag(S), 1)


def test_cholesky_textbook(O):
    rng = np.random.default_rng(0)
    for n in range(1, 8):
        A = rng.normal(size=(n, n))
        A = A @ A.T + n * np.eye(n)
        L = O.cholesky(A)
        assert np.allclose(L, np.linalg.cholesky(A), atol=1e-13)
    L2 = O.cholesky([[1, 0.707107], [0.707107, 1]])
    assert L2[1, 0] == pytest.approx(0.707107) and L2[1, 1] == pytest.approx(0.707107, abs=1e-6)
    with pytest.raises(np.linalg.LinAlgError):
        O.cholesky([[1, 2], [2, 1]])


def test_orthant_closed_forms(O):
    # n = 1: Phi
    assert O.mvn_orthant([1.0], [1.2]) == pytest.approx(special.ndtr(1.2), abs=1e-15)
    # n = 2 at the origin (Sheppard): 1/4 + asin(rho)/(2 pi), rho = sqrt(r2)
    for r2 in [0.05, 0.3, 0.5, 0.9]:
        exact = 0.25 + math.asin(math.sqrt(r2)) / (2 * math.pi)
        assert O.mvn_orthant([1, r2], [0, 0]) == pytest.approx(exact, abs=1e-12)
    # n = 3 at the origin: 1/8 + sum_{i<j} asin(rho_ij)/(4 pi); r=(1,.5,.25) gives 7/24
    assert O.mvn_orthant([1, 0.5, 0.25], [0, 0, 0]) == pytest.approx(7 / 24, abs=1e-12)
    r = [1, 0.6, 0.2]
    S = O.null_corr(r)
    exact = 0.125 + sum(math.asin(S[i, j]) for i, j in [(0, 1), (0, 2), (1, 2)]) / (4 * math.pi)
    assert O.mvn_orthant(r, [0, 0, 0]) == pytest.approx(exact, abs=1e-12)


def test_orthant_infinite_bound_marginalises(O):
    r = [1, 0.45, 0.15]
    a = O.mvn_orthant(r, [1.1, 2.0, math.inf])
    b = O.mvn_orthant(r[:2], [1.1, 2.0])
    assert a == pytest.approx(b, abs=1e-13)


def test_orthant_vs_one_dimensional_quad(O):
    # n = 3: X1 and X3 are independent given X2 (Markov), so
    # P = int phi(x) Phi((b1 - sqrt(r2) x)/sqrt(1-r2)) Phi((b3 - sqrt(r3/r2) x)/sqrt(1-r3/r2)) dx over x < b2.
    rng = np.random.default_rng(1)
    for _ in range(6):
        r2 = rng.uniform(0.1, 0.9)
        r3 = rng.uniform(0.05, 0.95) * r2
        b = rng.uniform(-1.5, 3.5, size=3)
        f = lambda x: (stats.norm.pdf(x) * special.ndtr((b[0] - math.sqrt(r2) * x) / math.sqrt(1 - r2))
                       * special.ndtr((b[2] - math.sqrt(r3 / r2) * x) / math.sqrt(1 - r3 / r2)))
        ref, _ = integrate.quad(f, -12, b[1], epsabs=1e-14, epsrel=1e-13, limit=200)
        assert O.mvn_orthant([1, r2, r3], b) == pytest.approx(ref, abs=1e-11)


def test_orthant_vs_genz_higher_n(O):
    # n = 5 against scipy's Genz integration (independent algorithm, tolerance 1e-8)
    r = [1.0, 0.8, 0.6, 0.4, 0.2]
    S = O.null_corr(r)
    b = np.array([2.0, 1.5, 2.2, 1.0, 2.5])
    ref = stats.multivariate_normal(mean=np.zeros(5), cov=S, abseps=1e-10, releps=1e-10, maxpts=10_000_000).cdf(b)
    assert O.mvn_orthant(r, b) == pytest.approx(ref, abs=2e-7)


def test_fwer_examples_and_monotone(O):
    assert O.fwer([1.0], [0.025]) == pytest.approx(0.025, abs=1e-15)
    # S:253 fwer(.0125,.0125; r2=.5) in (0.0125, 0.025), bivariate CDF by scipy
    S = O.null_corr([1, 0.5])
    z = special.ndtri(1 - 0.0125)
    ref = 1 - stats.multivariate_normal(mean=[0, 0], cov=S).cdf([z, z])
    val = O.fwer([1, 0.5], [0.0125, 0.0125])
    assert 0.0125 < val < 0.025 and val == pytest.approx(ref, abs=1e-7)
    # near-perfect correlation: tests coincide
    assert O.fwer([1, 1 - 1e-6], [0.025, 0.025]) == pytest.approx(0.025, abs=1e-4)
    # monotone in every alpha_i
    r = [1, 0.45, 0.15]
    base = [0.005, 0.01, 0.008]
    f0 = O.fwer(r, base)
    for i in range(3):
        a = list(base)
        a[i] += 1e-4
        assert O.fwer(r, a) > f0


def test_orthant_n4_close_ratios_vs_genz(O):
    """n = 4 with adjacent r ratios 0.99 (conditional sd 0.1): against scipy's Genz integration and the
    FWER bounds max(alpha) <= FWER <= sum(alpha) (the quadrature must follow the narrowest sd)."""
    r = [1.0, 0.99, 0.98, 0.97]
    S = O.null_corr(r)
    b = np.array([2.2, 2.0, 2.5, 1.9])
    ref = stats.multivariate_normal(mean=np.zeros(4), cov=S, abseps=1e-9, releps=1e-9, maxpts=20_000_000).cdf(b)
    assert O.mvn_orthant(r, b) == pytest.approx(ref, abs=2e-6)
    a = np.array([0.006, 0.006, 0.006, 0.006])
    f = O.fwer(r, a)
    assert a.max() < f < a.sum()
