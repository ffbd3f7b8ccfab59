"""C2 time-to-optimal-design in isolation (tuning harness; bench.py reports the same path in its line).

    python tools/tto_c2.py [--plan-first] [--reps 2] [--grid G]
Problem statement -> candidates (GPU alpha_n solve, N3 subsets) -> design init -> TPS plans (during the MC
pass unless --plan-first) -> one MC pass (1e6 draws/design) -> finalize -> TPS+GCV -> argmax -> per-problem
L-BFGS optimum; prints one JSON line per repetition with the phase times.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plan-first", action="store_true")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--grid", type=int, default=0, help="K1 persistent grid blocks (0: one tile per warp)")
    a = ap.parse_args()
    import torch
    from paper_2005_10494_b200 import mc
    from paper_2005_10494_b200 import workloads as W
    specs = W.c2_problems()
    for rep in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        probs = [mc.problem_formula10(s.r, s.delta0(), s.i3, s.alpha0) for s in specs]
        alpha, pod = mc.candidates(probs, m=W.GRID_M, n3=W.N3, seed=W.SEED)
        t1 = time.perf_counter()
        dsg = mc.Design(probs, alpha, pod, seed=W.SEED)
        dsg.set_launch(0, a.grid)
        dsg.smooth_plan(wait=a.plan_first)
        t2 = time.perf_counter()
        sums = dsg.new_sums()
        dsg.evaluate(sums, 0, W.DRAWS["C2"])
        mean, var = dsg.finalize(sums, W.DRAWS["C2"])
        sm, lam = dsg.smooth(mean, -1.0)
        idx, val, _ = dsg.argmax(sm, with_host=False)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        A, v, st = dsg.refine(mean, -1.0)
        t4 = time.perf_counter()
        dsg.close()
        print(json.dumps({"rep": rep, "plan_first": a.plan_first, "grid": a.grid, "candidates_s": t1 - t0, "init_plan_s": t2 - t1,
                          "mc_smooth_s": t3 - t2, "refine_s": t4 - t3, "total_s": t4 - t0}), flush=True)


if __name__ == "__main__":
    main()
