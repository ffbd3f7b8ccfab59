"""Time the TPS plan build (mc_smooth_plan) for k C2 problems (tuning harness; not the bench).

    python tools/time_plan.py 1 8 64
Prints one JSON line per k: seconds for candidates, design init and the plan."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2005_10494_b200 import mc
    from paper_2005_10494_b200 import workloads as W
    specs = W.c2_problems()
    for k in [int(x) for x in sys.argv[1:]] or [1, 8, 64]:
        sub = specs[:: max(1, len(specs) // k)][:k]
        probs = [mc.problem_formula10(s.r, s.delta0(), s.i3, s.alpha0) for s in sub]
        t0 = time.perf_counter()
        alpha, pod = mc.candidates(probs, m=W.GRID_M, n3=W.N3, seed=W.SEED)
        t1 = time.perf_counter()
        dsg = mc.Design(probs, alpha, pod, seed=W.SEED)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        dsg.smooth_plan()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(json.dumps({"problems": k, "designs": int(dsg.D), "candidates_s": t1 - t0, "init_s": t2 - t1,
                          "plan_s": t3 - t2, "plan_ms_per_problem": 1e3 * (t3 - t2) / k}), flush=True)
        dsg.close()


if __name__ == "__main__":
    main()
