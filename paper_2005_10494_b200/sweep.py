"""NEXT f2: choose the nested subpopulations r.

P:234: "First, we specify many settings of values of r, calculate their corresponding optimal powers
solved from problem (fopt).  Second, we fit TPS of optimal power as functions of r.  At last, we find
optimal solution of r on the fitted TPS using the same procedure as for the TPS P~(alpha)."
P:238: "the optimal design is defined by the optimal value of r together with optimal solution of alpha
under the setting of r".

Orchestration only: every numeric step runs in the C-ABI library (candidates, fused MC, all_reduce,
finalize, TPS smoothing, the L-BFGS optimum per problem, the host TPS over r and its maximum).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import mc


@dataclass
class SweepResult:
    r: np.ndarray            # [P, n-1] free cutoffs (r_2..r_n) of the lattice problems
    alpha_opt: np.ndarray    # [P, n] continuous optimum per problem (f1)
    power_opt: np.ndarray    # [P] P~ at the optimum
    status: np.ndarray       # [P] mc_refine status
    r_star: np.ndarray       # [n-1] maximiser of the TPS over r
    power_r_star: float      # the r-surface value at r*
    lambda_r: float


def optimal_powers(problems, m: int, n3: int, seed: int, total_samples: int, est: int = mc.EST_COND,
                   lam: float = -1.0, device: int = 0, rank: int = 0, world: int = 1):
    """Solve (fopt) for every problem: candidates -> MC -> TPS -> argmax start -> L-BFGS optimum."""
    alpha, pod = mc.candidates(problems, m=m, n3=n3, seed=seed, device=device)
    dsg = mc.Design(problems, alpha, pod, seed=seed, estimator=est, device=device)
    res = mc.evaluate_design_objective(dsg, total_samples, lam=lam, rank=rank, world=world)
    A, v, st = dsg.refine(res.mean, lam)
    dsg.close()
    return A, v, st


def sweep(problems, m: int, n3: int, seed: int, total_samples: int, est: int = mc.EST_COND,
          lam: float = -1.0, lam_r: float = -1.0, device: int = 0, rank: int = 0, world: int = 1) -> SweepResult:
    """Run the r-sweep over `problems` (one scenario: same prior law, different r)."""
    A, v, st = optimal_powers(problems, m, n3, seed, total_samples, est, lam, device, rank, world)
    n = problems[0].n
    r = np.array([[p.r[i] for i in range(1, n)] for p in problems])
    ok = st != 1
    surf = mc.Surface(r[ok], v[ok], lam_r)
    r_star, p_star = surf.maximum()
    return SweepResult(r=r, alpha_opt=A, power_opt=v, status=st, r_star=r_star, power_r_star=p_star,
                       lambda_r=surf.lam)
