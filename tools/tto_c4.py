"""C4 time-to-optimal-design, repeated (tuning harness for the C4 occupancy question).

    MC_LIB_PATH=tools/lib_X.so python tools/tto_c4.py [--reps 4]
Each repetition: candidates (256 strata problems x 256 alpha_1, alpha_2 solved) -> fused MC (1e6 draws) ->
finalize -> separable kernel smoother with GCV -> argmax; prints one JSON line per repetition (wall clock
from the problem statement to the optimum on the host) and the fused-kernel time alone (CUDA events)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=4)
    a = ap.parse_args()
    import torch
    from paper_2005_10494_b200 import mc, sweep
    from paper_2005_10494_b200 import workloads as W
    for rep in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g = sweep.c4_grid_optimum(W.c4_r2_values(), 211.0, W.C4_STRATA, W.C4_GRID, W.DRAWS["C4"], W.SEED)
        t1 = time.perf_counter()
        probs = [mc.problem_strata(r2, 211.0, W.C4_STRATA) for r2 in W.c4_r2_values()]
        alpha, pod = mc.candidates(probs, m=W.C4_GRID, n3=0, seed=W.SEED)
        dsg = mc.Design(probs, alpha, pod, seed=W.SEED)
        s = dsg.new_sums()
        dsg.evaluate(s, 0, W.DRAWS["C4"])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dsg.evaluate(s, 0, W.DRAWS["C4"])
        e1.record()
        torch.cuda.synchronize()
        dsg.close()
        print(json.dumps({"lib": os.environ.get("MC_LIB_PATH", "default"), "rep": rep, "tto_s": t1 - t0,
                          "kernel_ms": e0.elapsed_time(e1), "r2_star": g.r2}), flush=True)


if __name__ == "__main__":
    main()
