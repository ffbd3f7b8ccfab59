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


@dataclass
class GridOptimum:
    r2: float                # optimal cutoff of the (r2, alpha_1) grid
    alpha: np.ndarray        # [2] (alpha_1, alpha_2) at the optimum (alpha_2 solved)
    power_smoothed: float    # P~ at the optimum
    power_hat: float         # P^ there, and its standard error
    se: float
    bandwidths: tuple        # (h_r, h_alpha) chosen by GCV
    index: int               # design index (row-major r2 x alpha_1)
    smoothed: np.ndarray     # [nr, na] P~
    mean: np.ndarray         # [nr, na] P^


def c4_grid_optimum(r2_values, i3: float, strata, m: int, total_samples: int, seed: int, est: int = mc.EST_COND,
                    device: int = 0, rank: int = 0, world: int = 1) -> GridOptimum:
    """Configuration C4: the dense cutoff x allocation grid under the strata prior.
    One problem per cutoff r2, the m-point alpha_1 grid of each with alpha_2 solved (a1), the fused MC
    pass over all designs (a2-a8), the separable kernel smoother over (r2, alpha_1) (a9, R23) and the
    argmax (a10)."""
    torch = mc._torch()
    probs = [mc.problem_strata(r2, i3, strata) for r2 in r2_values]
    alpha, pod = mc.candidates(probs, m=m, n3=0, seed=seed, device=device)
    nr = len(probs)
    if len(alpha) != nr * m:
        raise RuntimeError(f"C4 grid: {len(alpha)} feasible designs, expected {nr * m}")
    dsg = mc.Design(probs, alpha, pod, seed=seed, estimator=est, device=device)
    try:
        res = mc.evaluate_design_objective(dsg, total_samples, smooth=False, rank=rank, world=world)
        grid = res.mean.view(nr, m)
        xr = np.asarray(r2_values, dtype=np.float64)
        xa = alpha[:m, 0].copy()
        sm, h = mc.grid_smooth(grid, xr, xa)
        _, _, (bi, bv) = dsg.argmax(sm.view(-1))
        mean = res.mean.cpu().numpy()
        se = float(np.sqrt(res.var[bi].item() / total_samples))
        return GridOptimum(r2=float(xr[bi // m]), alpha=alpha[bi].copy(), power_smoothed=bv, power_hat=float(mean[bi]),
                           se=se, bandwidths=h, index=bi, smoothed=sm.cpu().numpy(), mean=mean.reshape(nr, m))
    finally:
        dsg.close()
