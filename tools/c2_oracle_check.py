"""The north-star acceptance check on the FULL C2 grid run (tools/c2_full_run.py, 1e9 draws per design):
for a sample of problems, the ORACLE re-evaluates the GPU's top-K designs of each problem over the SAME
(design, sample) Philox streams at the run's full draw count, and the per-design estimates and the argmax
are compared (the C3 slice gets the same check inside bench.py, `c3_oracle_check`).

    python tools/c2_oracle_check.py gpurun_out/c2_1e9_r2.json [--problems 0,96,...] [--top 2] [--cores 6]
        > profiles/r02/c2_1e9_oracle_check.json

Designs: the oracle's own candidates (O.candidates, seed + problem index: the same alpha grid, alpha_3 within
1e-11 and the same subset as the GPU's mc.candidates); C2 has exactly N3 = 2000 designs per
problem, so problem k's local design i is global design 2000 k + i (the Philox key).  Test infrastructure:
reads the GPU run's JSON / npy output and calls only oracle/.
"""
import argparse
import json
import os
import sys
import time
from multiprocessing import get_context

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _worker(job):
    from oracle import oracle as O
    r, delta0, i3, alpha0, a, seed, design, s0, n = job
    prob = O.formula10_problem(r, delta0, i3, alpha0)
    return design, O.design_sums(prob, a, 0, seed, design, s0, n).tolist()


def _cands(k):
    from oracle import oracle as O
    from paper_2005_10494_b200 import workloads as W
    sp = W.c2_problems()[k]
    return O.candidates(sp.r, sp.alpha0, W.GRID_M, W.N3, W.SEED + k)


def _nice():
    try:
        os.nice(10)
    except OSError:
        pass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("run_json")
    ap.add_argument("--problems", default="", help="comma-separated problem indices (default: every 3rd sampled "
                                                   "problem of tests/golden/c2_exact_sample.json)")
    ap.add_argument("--top", type=int, default=2)
    ap.add_argument("--cores", type=int, default=max(1, (os.cpu_count() or 2) - 2))
    ap.add_argument("--draws", type=int, default=0, help="override the draw count (smoke runs only)")
    a = ap.parse_args()
    from oracle import oracle as O
    from paper_2005_10494_b200 import workloads as W
    O.build()
    run = json.load(open(a.run_json))
    mean = np.load(a.run_json.replace(".json", "_mean.npy"))
    N = a.draws or int(run["draws_per_design"])
    specs = W.c2_problems()
    assert run["designs"] == len(specs) * W.N3, "C2 has N3 designs per problem"
    if a.problems:
        probs = [int(x) for x in a.problems.split(",")]
    else:
        ex = json.load(open(os.path.join(ROOT, "tests", "golden", "c2_exact_sample.json")))
        probs = [e["problem"] for e in ex["problems"]][::3]
    gp = {r["problem"]: r for r in run["problems"]}
    sel, jobs = [], []
    bounds = [N * k // a.cores for k in range(a.cores + 1)]
    with get_context("spawn").Pool(min(a.cores, len(probs)), initializer=_nice) as pool:
        cands = pool.map(_cands, probs, chunksize=1)       # the oracle's alpha_3 bisections: minutes per problem
    for k, A in zip(probs, cands):
        sp = specs[k]
        m = mean[W.N3 * k: W.N3 * (k + 1)]
        order = np.argsort(-m, kind="stable")
        top = [int(i) for i in order[:a.top]]
        sel.append((k, top, A, m, order))
        for i in top:
            for c in range(a.cores):
                jobs.append((sp.r, sp.delta0(), sp.i3, sp.alpha0, A[i].tolist(), W.SEED, W.N3 * k + i, bounds[c],
                             bounds[c + 1] - bounds[c]))
    t0 = time.perf_counter()
    with get_context("spawn").Pool(a.cores, initializer=_nice) as pool:
        res = pool.map(_worker, jobs, chunksize=1)
    wall = time.perf_counter() - t0
    sums = {}
    for d, s in res:
        sums.setdefault(d, np.zeros(2, dtype=np.int64))
        sums[d] += np.array(s, dtype=np.int64)
    rows, worst, ident = [], 0.0, 0
    for k, top, A, m, order in sel:
        se = gp[k]["SE"]
        po = [float(O.finalize(sums[W.N3 * k + i], N)[0][0]) for i in top]
        pg = [float(m[i]) for i in top]
        rel = [abs(g - o) / o for g, o in zip(pg, po)]
        worst = max(worst, max(rel))
        max_abs = max(abs(g - o) for g, o in zip(pg, po))
        io = top[int(np.argmax(po))]
        unchecked = float(m[order[a.top]]) if len(order) > a.top else -1.0
        same = io == top[0]
        ident += same
        rows.append({"problem": k, "scenario": specs[k].scenario, "r": list(specs[k].r), "designs_checked": top,
                     "alpha": [[float(x) for x in A[i]] for i in top], "P_gpu": pg, "P_oracle": po, "rel_diff": rel,
                     "SE": se, "argmax_gpu": top[0], "argmax_oracle_among_checked": io, "argmax_identical": bool(same),
                     "gpu_run_raw_argmax": gp[k]["raw_argmax_local"],
                     "unchecked_gpu_max": unchecked,
                     "unchecked_cannot_win": bool(unchecked < max(po) - 2 * max_abs)})
    out = {"workload": "C2 full grid (513 problems x 2000 designs) at %.0e draws/design: sampled problems" % N,
           "draws_per_design": N, "problems_checked": len(rows), "top_k": a.top,
           "oracle_draws": float(N) * sum(len(t) for _, t, _, _, _ in sel), "oracle_wall_s": wall,
           "cores": a.cores, "max_rel_diff": worst, "tolerance": 1e-5, "pass_rel": worst <= 1e-5,
           "argmax_identical": ident, "rows": rows}
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
