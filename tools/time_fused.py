"""Time the fused MC kernel alone on a C2-shaped workload (tuning harness; not the bench).

    MC_LIB_PATH=/tmp/variant.so python tools/time_fused.py [--problems 6] [--est cond] [--threads 256]
Prints one JSON line: draws/s of mc_evaluate_grid (CUDA events, 2 warm-up + 5 timed launches).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problems", type=int, default=6)
    ap.add_argument("--est", default="cond")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--draws", type=int, default=1_000_000)
    ap.add_argument("--crn", action="store_true")
    ap.add_argument("--c4", action="store_true", help="time the C4 strata-prior kernel (model 1)")
    ap.add_argument("--crossed", type=str, default="", help="N1,N2: time the crossed estimator (IND ctx)")
    a = ap.parse_args()
    import torch
    from paper_2005_10494_b200 import mc
    from paper_2005_10494_b200 import workloads as W
    if a.c4:
        # C4 strata prior: 16 cutoffs x the 256-point alpha_1 grid
        probs = [mc.problem_strata(r2, 211.0, W.C4_STRATA) for r2 in W.c4_r2_values()[::16]]
        alpha, pod = mc.candidates(probs, m=W.C4_GRID, n3=0, seed=W.SEED)
    else:
        specs = W.c2_problems()[:: max(1, 513 // a.problems)][: a.problems]
        probs = [mc.problem_formula10(s.r, s.delta0(), s.i3, s.alpha0) for s in specs]
        alpha, pod = mc.candidates(probs, m=W.GRID_M, n3=W.N3, seed=W.SEED)
    dsg = mc.Design(probs, alpha, pod, seed=W.SEED, estimator=0 if a.est == "cond" else 1)
    dsg.set_launch(a.threads, a.grid)
    if a.crn:
        dsg.set_sampling(True)
    sums = dsg.new_sums()
    if a.crossed:
        n1, n2 = (int(x) for x in a.crossed.split(","))
        dsg.evaluate_crossed(sums, n1, n2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dsg.evaluate_crossed(sums, n1, n2)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"crossed": [n1, n2], "designs": dsg.D, "ms": ms,
                          "pairs_per_s": dsg.D * n1 * n2 / (ms * 1e-3)}), flush=True)
        return
    for _ in range(2):
        dsg.evaluate(sums, 0, a.draws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        dsg.evaluate(sums, 0, a.draws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"lib": mc.lib_path(), "est": a.est, "crn": a.crn, "threads": a.threads, "designs": dsg.D,
                      "ms": ms, "draws_per_s": dsg.D * a.draws / (ms * 1e-3)}), flush=True)


if __name__ == "__main__":
    main()
