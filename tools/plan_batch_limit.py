"""Probe the largest cusolverDnXsyevBatched batch the TPS plan accepts at the C2 size (N = 2000 sites,
m = 1997): builds the plans of the first P C2 problems in ONE batch (P <= MC_PLAN_BATCH) for each P given.

    python tools/plan_batch_limit.py 171 192 224 240 255 256
"""
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
    for P in [int(x) for x in sys.argv[1:]]:
        probs = [mc.problem_formula10(s.r, s.delta0(), s.i3, s.alpha0) for s in specs[:P]]
        alpha, pod = mc.candidates(probs, m=W.GRID_M, n3=W.N3, seed=W.SEED)
        dsg = mc.Design(probs, alpha, pod, seed=W.SEED)
        t0 = time.perf_counter()
        try:
            dsg.smooth_plan()
            torch.cuda.synchronize()
            res = "ok"
        except Exception as exc:          # noqa: BLE001 — the probe reports the library's status
            res = f"{type(exc).__name__}: {str(exc)[:120]}"
        print(json.dumps({"P": P, "result": res, "s": time.perf_counter() - t0}), flush=True)
        dsg.close()


if __name__ == "__main__":
    main()
