"""Pins for the oracle's crossed N1 x N2 estimator (Formula 7 literally; NEXT f3 (ii), reading R1)."""
import math

import numpy as np
import pytest


def _prob(O):
    r = [1.0, 0.45, 0.15]
    return r, O.formula10_problem(r, 0.8 - 0.6 * np.array(r), 211.0)


def test_crossed_matches_bruteforce_definition(O):
    # tiny case recomputed from the word stream by the definition (independent Python loop)
    r, prob = _prob(O)
    alpha = [0.004, 0.012, 0.01]
    n1, n2 = 6, 9
    s = O.design_sums_crossed(prob, alpha, 3, 5, n1, n2)
    z = O.thresholds(alpha)
    L0 = np.linalg.cholesky(O.null_corr(r))

    def normals(tag, s0, k):
        out = []
        for j in range(k // 2):
            wr = O.lib().or_word_tagged(3, 5, tag, s0 + 2 * j)
            wa = O.lib().or_word_tagged(3, 5, tag, s0 + 2 * j + 1)
            R = math.sqrt(-2 * math.log(1 - (wr & 0x7FFFFF) / 2 ** 23))
            a = 2 * math.pi * (wa & 0x7FFFFF) / 2 ** 23
            out += [R * math.cos(a), R * math.sin(a)]
        return np.array(out)
    X = [L0 @ normals(3, l * 4, 4)[:3] for l in range(n2)]
    c = []
    for k in range(n1):
        eps = normals(2, k * 4, 4)[:3]
        b = z - np.sqrt(np.array(r) * 211.0) * (prob.theta + prob.Lp @ eps)
        c.append(sum(int(np.any(x > b)) for x in X))
    assert s[0] == sum(c) and s[1] == sum(v * v for v in c)


def test_crossed_variance_exceeds_the_a2_bound(O):
    """SURVEY finding 5: the crossed pairs are dependent, so Var(P^) ~ Var_Delta(g)/N1, not <= 1/(4 N1 N2)
    (A.2).  Over 40 seeds at N1 = N2 = 200 the sample variance exceeds the A.2 bound 3x and agrees
    with the outer-draw variance estimate."""
    r, prob = _prob(O)
    alpha = [0.00175781, 0.01386719, 0.01278707]
    n1 = n2 = 200
    ests, vs = [], []
    for seed in range(40):
        m, v = O.finalize_crossed(O.design_sums_crossed(prob, alpha, seed, 0, n1, n2), n1, n2)
        ests.append(m[0]); vs.append(v[0])
    sv = np.var(ests, ddof=1)
    assert sv > 3 / (4 * n1 * n2)
    assert 0.4 < sv / (np.mean(vs) / n1) < 2.5
    exact = O.assurance_gaussian(prob, alpha)
    assert abs(np.mean(ests) - exact) < 5 * math.sqrt(sv / 40)
