"""Generate tests/golden/c1_oracle_1e4.txt from the ORACLE only (BASELINE configs[0]):
the 51 C1 designs (n = 2, r2 = (k+1)/52, scenario (c) Delta0 = 0.8 - 0.6 r, I3 = 211, alpha_1 = 0.0125,
alpha_2 solved by the oracle from Formula 2) and their COND integer sums over samples [0, 1e4) of the
(design, sample) Philox stream with the master seed, P^ = S1 / (N 2^23), and the oracle's argmax.
The C-ABI test (tests/c_abi/c1_abi.c) reads this file: one header line, then per design
    k r2 delta0_1 delta0_2 alpha_1 alpha_2 S1 S2 P_hat

    python tests/golden/make_c1_oracle.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2005_10494_b200 import workloads as W  # noqa: E402

N = 10_000


def main():
    specs, a1 = W.c1_problems()
    rows, P = [], []
    for k, s in enumerate(specs):
        a2 = O.solve_alpha_n(s.r, s.alpha0, [a1], 1e-14)
        prob = O.formula10_problem(s.r, s.delta0(), s.i3, s.alpha0)
        S = O.design_sums(prob, [a1, a2], 0, W.SEED, k, 0, N)
        p = O.finalize(S, N)[0][0]
        P.append(p)
        d0 = s.delta0()
        rows.append(f"{k} {float(s.r[1])!r} {float(d0[0])!r} {float(d0[1])!r} {float(a1)!r} {float(a2)!r} {int(S[0])} {int(S[1])} {float(p)!r}")
    best = O.argmax(np.array(P))
    out = os.path.join(ROOT, "tests", "golden", "c1_oracle_1e4.txt")
    with open(out, "w") as f:
        f.write(f"# C1 oracle (tests/golden/make_c1_oracle.py): designs {len(rows)} draws {N} seed {W.SEED} "
                f"i3 211 alpha0 0.025 argmax {best}\n")
        f.write("\n".join(rows) + "\n")
    print(out, "argmax", best)


if __name__ == "__main__":
    main()
