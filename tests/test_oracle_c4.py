"""Pins for the oracle's C4 strata-prior model (synthetic extension, not in the paper)."""
import math

import numpy as np
import pytest

from paper_2005_10494_b200 import workloads as W

SEED = W.SEED


def _mc(O, r2, sp, alpha, est, N, design=0):
    s = O.design_sums_strata(r2, 211.0, sp, alpha, est, SEED, design, 0, N)
    m, v = O.finalize(s, N)
    return float(m[0]), float(v[0])


def test_record_sizes_c4(O):
    assert O.record_uniforms(2, 5, 0) == 12 and O.record_words(2, 5, 0) == 10   # sample pair: 5 BM pairs + 2 SOV
    assert O.record_uniforms(2, 5, 1) == 16 and O.record_words(2, 5, 1) == 12   # 7 normals -> 4 pairs per sample


@pytest.mark.parametrize("est", [0, 1])
def test_zero_spread_is_exact_bivariate_orthant(O, est):
    # all five spreads 0: Delta is deterministic and P = 1 - Phi_2(z - mu; sqrt(r2)) exactly
    sp = np.array(W.C4_STRATA)
    sp[1::2] = 0.0
    r2 = 0.3
    a1 = 0.006
    a2 = O.solve_alpha_n([1, r2], 0.025, [a1])
    z = O.thresholds([a1, a2])
    b = O.strata_b(r2, 211.0, sp, z, np.zeros(5))
    exact = 1 - O.mvn_orthant([1, r2], b)
    N = 100_000
    m, v = _mc(O, r2, sp, [a1, a2], est, N)
    assert abs(m - exact) < 5 * math.sqrt(v / N) + 1e-12
    # the deterministic prior mean at pi = 0.35 > r2 = 0.3: responders cover the whole subset (q+ = 1)
    assert b[1] == pytest.approx(z[1] - math.sqrt(0.3 * 211.0 * 0.9) * 0.6, rel=1e-12)


@pytest.mark.parametrize("r2,a1", [(0.3, 0.005), (0.7, 0.0125)])
def test_mc_matches_tensor_quadrature(O, r2, a1):
    # Gauss-Hermite over four components x Gauss-Legendre on both sides of the prevalence kink
    sp = np.array(W.C4_STRATA)
    a2 = O.solve_alpha_n([1, r2], 0.025, [a1])
    quad = O.assurance_strata_quadrature(r2, 211.0, sp, [a1, a2], n_gh=6, n_gl=16)
    N = 200_000
    for est in (0, 1):
        m, v = _mc(O, r2, sp, [a1, a2], est, N, design=est)
        assert abs(m - quad) < 5 * math.sqrt(v / N) + 2e-4, (est, m, quad)


def test_strata_b_kink_and_monotonicity(O):
    # q+ = min(1, pi/r2) bends at pi = r2; b_2 (subset threshold) decreases as the effect+ increases
    sp = np.array(W.C4_STRATA)
    z = np.array([2.5, 2.2])
    e = np.zeros(5)
    b0 = O.strata_b(0.5, 211.0, sp, z, e)
    e[1] = 1.0
    b1 = O.strata_b(0.5, 211.0, sp, z, e)
    assert b1[1] < b0[1] and b1[0] < b0[0]


@pytest.mark.parametrize("r2", [0.25, 0.6])
def test_gaussian_effects_reduce_to_bivariate_normal(O, r2):
    """An independent pin of the C4 mapping: with prevalence, variance and dropout held at
    their means (spreads 0) and only the two effects Gaussian, Delta = (Delta_1, Delta_2) is a linear map of
    (delta+, delta-), so Formula 4 is 1 - Phi_2(z; c E[Delta], Sigma0 + C Cov(Delta) C) — evaluated here by
    scipy's bivariate normal CDF from the mapping restated by hand, against the oracle's MC and its tensor
    quadrature.  r2 = 0.25 < pi = 0.35 (q+ = 1, q- > 0) and r2 = 0.6 > pi (q+ < 1, q- = 0)."""
    from scipy import stats
    sp = np.array(W.C4_STRATA, dtype=float)
    sp[1] = sp[7] = sp[9] = 0.0                       # logit pi, log v, logit d fixed
    pi = 1 / (1 + math.exp(-sp[0]))
    v = math.exp(sp[6])
    d = 1 / (1 + math.exp(-sp[8]))
    ieff = 211.0 * (1 - d) / v
    qp, qm = min(1.0, pi / r2), max(0.0, (pi - r2) / (1 - r2))
    A = np.array([[r2 * qp + (1 - r2) * qm, r2 * (1 - qp) + (1 - r2) * (1 - qm)],
                  [qp, 1 - qp]])
    mean_d = A @ np.array([sp[2], sp[4]])
    cov_d = A @ np.diag([sp[3] ** 2, sp[5] ** 2]) @ A.T
    c = np.sqrt(np.array([1.0, r2]) * ieff)
    a1 = 0.006
    a2 = O.solve_alpha_n([1, r2], 0.025, [a1])
    z = O.thresholds([a1, a2])
    S0 = np.array([[1.0, math.sqrt(r2)], [math.sqrt(r2), 1.0]])
    cov = S0 + np.diag(c) @ cov_d @ np.diag(c)
    exact = 1 - stats.multivariate_normal(mean=c * mean_d, cov=cov, abseps=1e-12, releps=1e-12).cdf(z)
    quad = O.assurance_strata_quadrature(r2, 211.0, sp, [a1, a2], n_gh=12, n_gl=8)
    assert quad == pytest.approx(exact, abs=2e-6)
    N = 200_000
    for est in (0, 1):
        m, var = _mc(O, r2, sp, [a1, a2], est, N, design=est + 3)
        assert abs(m - exact) < 5 * math.sqrt(var / N) + 1e-9, (est, m, exact)
