"""Exact reference for the C2 full-grid run (tools/c2_full_run.py), from the ORACLE only: for a sample of
the 513 C2 problems, the oracle's own candidate designs (m = 64 grid, alpha_3 by bisection, the seeded
N3 = 2000 subset with seed + problem index) and the exact Formula-4 value of every design
(Gaussian collapse + Markov orthant quadrature), its exact argmax and the top-2 gap.

    python tests/golden/make_c2_exact_sample.py --every 16 --max-r2 0.7

Test infrastructure: a committed script that calls only oracle/ (and the input generators) and writes the
stored expected values tests/golden/c2_exact_sample.{json,npz}; the GPU result of tools/c2_full_run.py is
compared with them by tools/c2_compare.py.
"""
import argparse
import json
import os
import sys
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def one(k):
    import oracle.oracle as O
    from paper_2005_10494_b200 import workloads as W
    sp = W.c2_problems()[k]
    A = O.candidates(sp.r, sp.alpha0, W.GRID_M, W.N3, W.SEED + k)
    prob = O.formula10_problem(sp.r, sp.delta0(), sp.i3, sp.alpha0)
    P = np.array([O.assurance_gaussian(prob, a) for a in A])
    order = np.argsort(-P, kind="stable")
    return {"problem": k, "scenario": sp.scenario, "r": list(sp.r), "designs": len(A),
            "exact_argmax_local": int(O.argmax(P)), "exact_max": float(P.max()),
            "alpha_argmax": [float(x) for x in A[O.argmax(P)]],
            "top5_local": [int(i) for i in order[:5]], "top5_P": [float(P[i]) for i in order[:5]],
            "gap12": float(P[order[0]] - P[order[1]]), "P": P}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--every", type=int, default=16)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c2_exact_sample.json"))
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 4)
    ap.add_argument("--max-r2", type=float, default=0.7,
                    help="skip problems with r2 above this (the oracle's FWER quadrature needs ~1 h per problem "
                         "of 4096 bisection solves as rho -> 1)")
    a = ap.parse_args()
    from paper_2005_10494_b200 import workloads as W
    specs = W.c2_problems()
    ks = [k for k in range(0, 513, a.every) if specs[k].r[1] <= a.max_r2]
    with Pool(a.procs) as pool:
        rows = pool.map(one, ks)
    np.savez_compressed(a.out.replace(".json", ".npz"), **{f"P{r['problem']}": r.pop("P") for r in rows})
    with open(a.out, "w") as f:
        json.dump({"source": "oracle only (tests/golden/make_c2_exact_sample.py)", "problems": rows}, f, indent=1)
    print(len(rows), "problems ->", a.out)


if __name__ == "__main__":
    main()
