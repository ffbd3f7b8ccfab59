"""Seeded synthetic workloads (BASELINE.json configs).

This module holds INPUTS only — problem lists, lattices, scenario laws and seeds as the
paper states them.  It contains none of the method's arithmetic (no thresholds, priors,
FWER solves or estimators), so it may serve both the CUDA path and the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

SEED = 0x0000002005105494          # the arXiv id; Philox key = (lo, hi)
FRESH_SEED = SEED ^ 0x00F1F1F100F1F1F1   # f1: fresh draws at the continuous optimum alpha* (independent key)
ALPHA0 = 0.025                      # P:221 / P:255, one-sided 0.025 (reading R9)
GRID_M = 64                         # candidate alpha grid per free dimension (reading R10)
N3 = 2000                           # P:221 / P:308 "N3 = 2000 random selected values of alpha"

# Sec. 3: Delta0_i = intercept + slope * r_i, I3 from Eq. 9 as printed.
SCENARIOS = {
    "a": {"intercept": 0.25, "slope": 0.0, "i3": 127.0},   # no biomarker effect
    "b": {"intercept": 0.30, "slope": -0.1, "i3": 211.0},  # weak biomarker effect
    "c": {"intercept": 0.80, "slope": -0.6, "i3": 211.0},  # strong biomarker effect
}


@dataclass(frozen=True)
class ProblemSpec:
    """One fixed-r problem as the paper states it: r, scenario law, I3, alpha0."""
    r: tuple
    scenario: str
    i3: float
    alpha0: float = ALPHA0

    def delta0(self):
        s = SCENARIOS[self.scenario]
        return tuple(s["intercept"] + s["slope"] * ri for ri in self.r)


def r_lattice(step: float = 0.05):
    """all (r2, r3) on the step grid of (0,1)^2 with 1 > r2 > r3 > 0 (171 for 0.05)."""
    k = int(round(1.0 / step))
    vals = [round(i * step, 10) for i in range(1, k)]
    return [(a, b) for a in vals for b in vals if a > b]


def c1_problems():
    """C1: n = 2 cutoff grid, r2 = (k+1)/52, k = 0..50, scenario (c), I3 = 211; alpha_1 = 0.0125
    and alpha_2 solved from Formula 2 (each side solves it with its own code)."""
    return [ProblemSpec(r=(1.0, (k + 1) / 52.0), scenario="c", i3=211.0) for k in range(51)], 0.0125


def c2_problems():
    """C2: 3 scenarios x 171 (r2, r3) pairs = 513 problems."""
    out = []
    for sc in ("a", "b", "c"):
        for r2, r3 in r_lattice(0.05):
            out.append(ProblemSpec(r=(1.0, r2, r3), scenario=sc, i3=SCENARIOS[sc]["i3"]))
    return out


def c2_slice():
    """C2/C3 headline slice: scenario (c), r = (1, 0.45, 0.15), all valid m = 64 designs."""
    return ProblemSpec(r=(1.0, 0.45, 0.15), scenario="c", i3=211.0)


def c5_problem(n: int):
    """C5: r_i = (n - i + 1)/n, scenario (c), I3 = 211."""
    return ProblemSpec(r=tuple((n - i) / n for i in range(n)), scenario="c", i3=211.0)


def n4_problem():
    """The paper's n = 4 workload (N3 = 4000, d = 3 TPS): scenario (c) law, I3 = 211, nested
    fractions r = (1, 0.6, 0.35, 0.15) (the paper does not print its n = 4 r; these are a lattice point)."""
    return ProblemSpec(r=(1.0, 0.6, 0.35, 0.15), scenario="c", i3=211.0)


N4_GRID_M = 32      # m^3 = 32768 grid points over (alpha_1, alpha_2, alpha_3), alpha_4 solved
N4_N3 = 4000


# draws per design (BASELINE.json configs)
DRAWS = {"C1": 10_000, "C2": 1_000_000, "C3": 1_000_000_000, "C4": 1_000_000, "C5": 1_000_000}


# C4: synthetic 5-D strata prior (not in the paper), n = 2, dense 256 x 256 design grid
# r2 = (i + 1/2)/256 x alpha_1 = (j + 1/2) alpha0/256 (alpha_2 solved), I3 = 211.
# (mean, sd) of: logit prevalence, effect+, effect-, log variance, logit dropout.
import math as _math

C4_STRATA = (_math.log(0.35 / 0.65), 0.4, 0.6, 0.15, 0.05, 0.10, 0.0, 0.2, _math.log(0.1 / 0.9), 0.5)
C4_GRID = 256


def c4_r2_values(m: int = C4_GRID):
    return [(i + 0.5) / m for i in range(m)]
