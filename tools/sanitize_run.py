"""A small pass over every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
Candidates (n = 3 warp kernel, n = 4 chain CTAs), fused K1 (COND/IND, steady and masked tiles, n = 1..4 and the
C4 strata model), CRN, crossed, finalize, TPS plan (batched and Dsyevd lanes) + smoothing + refine, the C4 grid
smoother (own DGEMM), argmax, the dump hooks."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2005_10494_b200 import mc
    from paper_2005_10494_b200 import workloads as W
    specs = W.c2_problems()[::100][:5]
    probs = [mc.problem_formula10(s.r, s.delta0(), s.i3, s.alpha0) for s in specs]
    alpha, pod = mc.candidates(probs, m=12, n3=60, seed=W.SEED)
    for est in (mc.EST_COND, mc.EST_IND):
        dsg = mc.Design(probs, alpha, pod, seed=W.SEED, estimator=est)
        s = dsg.new_sums()
        dsg.evaluate(s, 0, 10_000)            # steady tiles + a masked tail
        dsg.evaluate(s, 2**32 - 3000, 6000)   # across the 32-bit block-counter wrap
        mean, var = dsg.finalize(s, 16_000)
        sm, lam = dsg.smooth(mean, -1.0)
        dsg.argmax(sm)
        dsg.refine(mean, -1.0)
        dsg.draw_dump(torch.zeros(8, dtype=torch.int64).cuda(), torch.arange(8).cuda())
        dsg.set_sampling(True)
        dsg.evaluate(s, 0, 5000)
        dsg.close()
    dx = mc.Design(probs[:1], alpha[pod == 0], np.zeros(int((pod == 0).sum()), dtype=np.int32), seed=1,
                   estimator=mc.EST_IND)
    sx = dx.new_sums()
    dx.evaluate_crossed(sx, 512, 1024)
    dx.finalize_crossed(sx, 512, 1024)
    dx.close()
    # n = 1, 2, 4 and the chain FWER / explicit points
    for n in (1, 2, 4):
        sp = W.c5_problem(n)
        p = mc.problem_formula10(sp.r, sp.delta0(), sp.i3, sp.alpha0)
        A, pd = mc.candidates([p], m=6 if n == 4 else 16, n3=0, seed=1)
        mc.fwer(p, A[:4])
        d = mc.Design([p], A, pd, seed=3)
        s = d.new_sums()
        d.evaluate(s, 0, 4096 + 17)
        m, _ = d.finalize(s, 4096 + 17)
        if n >= 2:
            d.smooth(m, -1.0)
        d.close()
    A, ok = mc.solve_alpha_n([mc.problem_formula10([1.0, 0.6, 0.35, 0.15], [0.3] * 4, 211.0)],
                             np.full((3, 4), 0.003), np.zeros(3, dtype=np.int32))
    # C4 strata model + the grid smoother
    r2s = W.c4_r2_values(16)
    ps = [mc.problem_strata(r2, 211.0, W.C4_STRATA) for r2 in r2s]
    A4, pod4 = mc.candidates(ps, m=16, n3=0, seed=1)
    d4 = mc.Design(ps, A4, pod4, seed=1)
    s4 = d4.new_sums()
    d4.evaluate(s4, 0, 4096)
    m4, _ = d4.finalize(s4, 4096)
    mc.grid_smooth(m4.view(16, 16), np.array(r2s), A4[:16, 0])
    d4.close()
    torch.cuda.synchronize()
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
