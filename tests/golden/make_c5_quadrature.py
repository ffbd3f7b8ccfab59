"""Generate tests/golden/c5_quadrature.json from the ORACLE only (BASELINE configs[4], SURVEY §8(d) C5:
"dimension-independent MC error vs quadrature").

For n = 3..10 (r_i = (n-i+1)/n, scenario (c), I3 = 211, alpha_1 = 0.0125, alpha_2..alpha_n equal and solved
from Formula 2 by bisection): the exact Formula-4 value (Gaussian collapse + Markov transfer quadrature)
and the midpoint tensor-grid quadrature of the same expectation over the n-D prior (standardised
coordinates on [-5, 5]^n, m = floor(B^(1/n)) midpoints per axis, B = 4096 nodes budget, P:131's "standard
numerical integration" at a fixed budget), with its absolute error.

    python tests/golden/make_c5_quadrature.py
"""
import json
import math
import os
import sys
from itertools import product
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
BUDGET = 4096


def one(n):
    import oracle.oracle as O
    from paper_2005_10494_b200 import workloads as W
    spec = W.c5_problem(n)
    prob = O.formula10_problem(spec.r, spec.delta0(), spec.i3, spec.alpha0)
    a1, lo, hi = 0.0125, 0.0, 0.025
    for _ in range(40):
        mid = 0.5 * (lo + hi)
        if O.fwer(spec.r, [a1] + [mid] * (n - 1)) > 0.025:
            hi = mid
        else:
            lo = mid
    alpha = [a1] + [lo] * (n - 1)
    exact = O.assurance_gaussian(prob, alpha)
    z = O.thresholds(alpha)
    c = np.sqrt(np.asarray(spec.r) * spec.i3)
    m = int(math.floor(BUDGET ** (1.0 / n) + 1e-9))
    h = 10.0 / m
    grid = -5.0 + h * (np.arange(m) + 0.5)
    wts = np.exp(-0.5 * grid * grid) / math.sqrt(2 * math.pi) * h
    total, wsum = 0.0, 0.0
    for idx in product(range(m), repeat=n):
        eps = grid[list(idx)]
        w = float(np.prod(wts[list(idx)]))
        delta = prob.theta + prob.Lp @ eps
        total += w * (1.0 - O.mvn_orthant(spec.r, z - c * delta))
        wsum += w
    return {"n": n, "alpha": alpha, "exact": exact, "m": m, "nodes": m ** n, "quadrature": total,
            "abs_error": abs(total - exact), "weight_sum": wsum}


def main():
    with Pool(min(8, os.cpu_count() or 4)) as pool:
        rows = pool.map(one, range(3, 11))
    with open(os.path.join(HERE, "c5_quadrature.json"), "w") as f:
        json.dump({"source": "oracle only (tests/golden/make_c5_quadrature.py)", "budget_nodes": BUDGET,
                   "rows": rows}, f, indent=1)
    for r in rows:
        print(r["n"], r["m"], r["nodes"], "%.3e" % r["abs_error"])


if __name__ == "__main__":
    main()
