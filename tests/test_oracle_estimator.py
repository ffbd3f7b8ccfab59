"""Pins for the oracle's Monte-Carlo estimator (Formulas 4-7, A.2) against exact values."""
import math

import numpy as np
import pytest
from scipy import special

SEED = 0x0000002005105494


def _mc(O, prob, alpha, est, N, design=0, seed=SEED):
    sums = O.design_sums(prob, alpha, est, seed, design, 0, N)
    mean, var = O.finalize(sums, N)
    return float(mean[0]), float(var[0])


def test_point_mass_n1_is_exact_power(O):
    # Point-mass prior, n = 1, COND: every draw's u equals Phi(c theta - z) exactly.
    i3 = O.information_units(0.025, 0.1, 0.25)     # Eq. 9, exact
    theta = -math.log(1 - 0.25)
    prob = O.point_mass_problem([1.0], [theta], i3)
    for s in range(50):
        u = O.draw(prob, [0.025], O.EST_COND, SEED, 0, s)["u"]
        assert u == pytest.approx(0.9, abs=1e-12)   # Eq. 9 is built for power 1 - beta = 0.9
    mean, var = _mc(O, prob, [0.025], O.EST_COND, 1000)
    assert mean == pytest.approx(0.9, abs=2 ** -23)
    assert var < 1e-12


def test_sov_degenerate_thresholds(O):
    r = [1, 0.45, 0.15]
    prob = O.point_mass_problem(r, [0.0, 0.0, 0.0], 211.0)
    # alpha = 0 everywhere: z = +inf, no test can reject -> u = 0 for both estimators
    for est in (O.EST_COND, O.EST_IND):
        mean, _ = _mc(O, prob, [0.0, 0.0, 0.0], est, 200)
        assert mean == 0.0
    # huge effect: every b_i -> -inf, u = 1
    prob2 = O.point_mass_problem(r, [50.0, 50.0, 50.0], 211.0)
    for est in (O.EST_COND, O.EST_IND):
        mean, _ = _mc(O, prob2, [0.01, 0.01, 0.01], est, 200)
        assert mean == 1.0


@pytest.mark.parametrize("est", [0, 1])
def test_point_mass_at_null_gives_fwer(O, est):
    # Under H0 (theta = 0, point mass) the power is the FWER: Formula 2 vs Formula 4.
    r = [1, 0.45, 0.15]
    alpha = [0.006, 0.011, 0.009]
    prob = O.point_mass_problem(r, [0.0, 0.0, 0.0], 211.0)
    N = 200_000
    mean, var = _mc(O, prob, alpha, est, N)
    exact = O.fwer(r, alpha)
    assert abs(mean - exact) < 5 * math.sqrt(var / N)


@pytest.mark.parametrize("est", [0, 1])
def test_c1_designs_match_closed_form(O, est):
    # C1 (n=2 cutoff grid, Formula-10 prior, scenario (c)): MC within 5 SE of the Gaussian collapse.
    N = 20_000
    for k in [0, 13, 25, 50]:
        r = [1.0, (k + 1) / 52]
        a2 = O.solve_alpha_n(r, 0.025, [0.0125])
        prob = O.formula10_problem(r, 0.8 - 0.6 * np.array(r), 211.0)
        mean, var = _mc(O, prob, [0.0125, a2], est, N, design=k)
        exact = O.assurance_gaussian(prob, [0.0125, a2])
        assert abs(mean - exact) < 5 * math.sqrt(var / N), (k, mean, exact)


def test_cond_has_lower_variance_than_ind(O):
    # Rao-Blackwellisation: E[u_COND] = E[u_IND] but Var_COND <= Var_IND (reading R6)
    r = [1, 0.45, 0.15]
    prob = O.formula10_problem(r, 0.8 - 0.6 * np.array(r), 211.0)
    alpha = [0.00175781, 0.01386719, 0.01278707]
    _, v_cond = _mc(O, prob, alpha, O.EST_COND, 50_000)
    _, v_ind = _mc(O, prob, alpha, O.EST_IND, 50_000)
    assert v_cond < v_ind


def test_brute_force_quadrature_general_prior(O):
    # A non-Formula-10 Gaussian prior (independent components, different sd): no collapse to
    # a Markov orthant.  Brute force: Gauss-Hermite over Delta (2-D tensor) x exact orthant.
    r = [1.0, 0.4]
    theta = np.array([0.25, 0.45])
    cov = np.diag([0.03, 0.08])
    prob = O.Problem(r=np.array(r), i3=127.0, alpha0=0.025, theta=theta, prior_cov=cov)
    alpha = [0.01, O.solve_alpha_n(r, 0.025, [0.01])]
    z = np.array([O.threshold(a) for a in alpha])
    c = np.sqrt(np.array(r) * 127.0)
    x, w = np.polynomial.hermite_e.hermegauss(40)
    w = w / w.sum()
    L = np.linalg.cholesky(cov)
    exact = 0.0
    for i in range(40):
        for j in range(40):
            d = theta + L @ np.array([x[i], x[j]])
            exact += w[i] * w[j] * (1 - O.mvn_orthant(r, z - c * d))
    N = 100_000
    for est in (O.EST_COND, O.EST_IND):
        mean, var = _mc(O, prob, alpha, est, N, design=3)
        assert abs(mean - exact) < 5 * math.sqrt(var / N)


def test_variance_bound_appendix_a2(O):
    # A.2 with independent joint draws: Var(P^) = Var(u)/N <= 1/(4N).
    # Sample variance of P^ over 100 seeds must be <= 2 var_d / N (slack for chi-square noise).
    r = [1, 0.4]
    prob = O.formula10_problem(r, 0.3 - 0.1 * np.array(r), 211.0)
    alpha = [0.016, O.solve_alpha_n(r, 0.025, [0.016])]
    N = 2000
    est_vals, vars_ = [], []
    for seed in range(1, 101):
        m, v = _mc(O, prob, alpha, O.EST_IND, N, seed=seed)
        est_vals.append(m)
        vars_.append(v)
    sv = np.var(est_vals, ddof=1)
    assert sv <= 2 * np.mean(vars_) / N <= 2 / (4 * N)
    assert max(vars_) <= 0.25 * N / (N - 1) + 1e-12


def test_sums_are_additive_over_sample_ranges(O):
    # The integer sums of [0, N) equal the sums of any split: launch-shape free.
    r = [1, 0.45, 0.15]
    prob = O.formula10_problem(r, 0.8 - 0.6 * np.array(r), 211.0)
    alpha = [0.002, 0.0135, 0.0133]
    whole = O.design_sums(prob, alpha, 0, SEED, 11, 0, 1000)
    parts = sum(O.design_sums(prob, alpha, 0, SEED, 11, a, b - a) for a, b in [(0, 1), (1, 333), (333, 1000)])
    assert np.array_equal(whole, parts)
