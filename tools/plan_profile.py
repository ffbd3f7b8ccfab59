"""Time the TPS plan (row a9 prep) and the candidates (a1) of the C2 workload in isolation (tuning harness).

    python tools/plan_profile.py [--problems 64]
Prints one JSON line: seconds for mc_candidates and mc_smooth_plan (host wall clock around synchronising
calls) and per problem."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problems", type=int, default=64)
    a = ap.parse_args()
    import torch
    from paper_2005_10494_b200 import mc
    from paper_2005_10494_b200 import workloads as W
    specs = W.c2_problems()[: a.problems]
    probs = [mc.problem_formula10(s.r, s.delta0(), s.i3, s.alpha0) for s in specs]
    mc.candidates(probs[:2], m=W.GRID_M, n3=W.N3, seed=W.SEED)          # warm-up (context, module load)
    t0 = time.perf_counter()
    alpha, pod = mc.candidates(probs, m=W.GRID_M, n3=W.N3, seed=W.SEED)
    t1 = time.perf_counter()
    dsg = mc.Design(probs, alpha, pod, seed=W.SEED)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dsg.smooth_plan()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    vals = torch.full((dsg.D,), 0.9, dtype=torch.float64, device="cuda")
    dsg.smooth(vals, -1.0)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    for _ in range(3):
        dsg.smooth(vals, -1.0)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(json.dumps({"problems": len(probs), "designs": int(dsg.D), "candidates_s": t1 - t0, "plan_s": t3 - t2,
                      "plan_ms_per_problem": (t3 - t2) * 1e3 / len(probs), "smooth_ms": (t5 - t4) * 1e3 / 3}))


if __name__ == "__main__":
    main()
