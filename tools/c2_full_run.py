"""The north-star target run: the full paper-shaped 3-D design grid (C2: 513 problems x 2000 designs)
at >= 1e9 draws per design on one B200, in resumable chunks (one gpurun call each).

    python tools/c2_full_run.py --total 1000000000 --chunk 200000000 --ckpt runs/c2_1e9 --out gpurun_out/c2_1e9

Each call adds `chunk` draws per design to the integer sums of the checkpoint (samples [done, done+chunk)
of every design's own Philox stream) and saves it: the sums are exact integers, so the chunked run is
bit-identical to one uninterrupted pass.  The call that reaches `total` finalises: mean / SE per design,
TPS + GCV per problem, raw and smoothed argmax per problem, the L-BFGS optimum (f1), and writes
<out>.json (per problem) and <out>_mean.npy.  Product path only (no oracle).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--total", type=int, default=1_000_000_000)
    ap.add_argument("--chunk", type=int, default=200_000_000)
    ap.add_argument("--ckpt", default=os.path.join(ROOT, "runs", "c2_1e9"))
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c2_1e9"))
    a = ap.parse_args()
    import torch
    from paper_2005_10494_b200 import mc
    from paper_2005_10494_b200 import workloads as W

    specs = W.c2_problems()
    probs = [mc.problem_formula10(s.r, s.delta0(), s.i3, s.alpha0) for s in specs]
    alpha, pod = mc.candidates(probs, m=W.GRID_M, n3=W.N3, seed=W.SEED)
    dsg = mc.Design(probs, alpha, pod, seed=W.SEED)
    sums = dsg.new_sums()
    done, kernel_s = 0, 0.0
    if os.path.exists(a.ckpt + ".npz"):
        s, done, seed, meta = mc.checkpoint_load(a.ckpt)
        assert seed == W.SEED and s.shape == tuple(sums.shape), "checkpoint does not match the workload"
        sums.copy_(torch.from_numpy(s))
        kernel_s = float(meta.get("kernel_s", 0.0))
    count = min(a.chunk, a.total - done)
    if count > 0:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        dsg.evaluate(sums, done, count)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        kernel_s += ms / 1e3
        done += count
        os.makedirs(os.path.dirname(a.ckpt), exist_ok=True)
        mc.checkpoint_save(a.ckpt, sums, done, W.SEED, {"kernel_s": kernel_s, "designs": int(dsg.D)})
        print(json.dumps({"chunk_draws_per_design": count, "done": done, "chunk_s": ms / 1e3,
                          "draws_per_s": dsg.D * count / (ms / 1e3)}), flush=True)
    if done < a.total:
        return
    mean, var = dsg.finalize(sums, done)
    dsg.smooth_plan()
    sm, lam = dsg.smooth(mean, -1.0)
    idx_raw, val_raw, (bi, bv) = dsg.argmax(mean)
    idx_sm, val_sm, _ = dsg.argmax(sm)
    A_opt, v_opt, st = dsg.refine(mean, -1.0)
    m = mean.cpu().numpy()
    se = np.sqrt(var.cpu().numpy() / done)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    np.save(a.out + "_mean.npy", m)
    begin = np.searchsorted(pod, np.arange(len(specs)))
    rows = []
    for k, sp in enumerate(specs):
        ir, ism = int(idx_raw[k]), int(idx_sm[k])
        rows.append({"problem": k, "scenario": sp.scenario, "r": list(sp.r), "raw_argmax_local": ir - int(begin[k]),
                     "raw_alpha": [float(x) for x in alpha[ir]], "P_hat": float(m[ir]), "SE": float(se[ir]),
                     "smoothed_argmax_local": ism - int(begin[k]), "P_smoothed": float(val_sm[k]),
                     "lambda": float(lam[k]), "alpha_opt": [float(x) for x in A_opt[k]], "P_opt": float(v_opt[k]),
                     "refine_status": int(st[k])})
    out = {"workload": "C2 full: 513 problems x 2000 designs", "designs": int(dsg.D), "draws_per_design": done,
           "total_draws": float(dsg.D) * done, "kernel_s": kernel_s,
           "draws_per_s": float(dsg.D) * done / kernel_s, "best_overall": [int(bi), float(bv)], "problems": rows}
    with open(a.out + ".json", "w") as f:
        json.dump(out, f)
    print(json.dumps({k: out[k] for k in ("designs", "draws_per_design", "kernel_s", "draws_per_s")}), flush=True)


if __name__ == "__main__":
    main()
