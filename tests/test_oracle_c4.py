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
