#!/usr/bin/env python
"""Benchmark of the Monte-Carlo design-objective hot path (BASELINE.json metric: MC draws/s).

One step = one pass of rows a2-a10 over the whole workload: the fused MC kernel over
every design for this rank's sample shard, the int64 all_reduce (N > 1), finalize, TPS+GCV
smoothing per problem, and the per-problem argmax.  Design prep (row a1: candidates on the GPU,
thresholds, TPS plan) is done once before timing; inputs are resident in HBM when timing starts.

Default workload (BASELINE.json configs[1]): the paper's 3-D problem, 3 scenarios x
171 (r2, r3) cutoff pairs = 513 problems x N3 = 2000 candidate alpha designs = 1,026,000 designs,
1e6 draws per design (1.026e12 draws per step), sharded over ranks by Philox sample range.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--est cond|ind]
Multi-GPU: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2005_10494_b200 import workloads as W  # noqa: E402

# Per-draw issue slots of the fused kernel's steady-state loop (n = 3), counted from the sm_100a SASS
# of the library being timed by tools/sass_count.py: the ALU/issue roofline's work per
# draw.  The fallback constants are that tool's output for the committed kernel.
ISSUE_PER_DRAW_FALLBACK = {"cond": 112.5, "ind": 108.0}
PIPE_MIX_FALLBACK = {"cond": {"issue": 112.5, "fp32": 78.5, "sfu": 14.0, "imad_wide": 18.0},
                     "ind": {"issue": 108.0, "fp32": 26.0, "sfu": 12.0, "imad_wide": 27.0}}


def pipe_mix(est: str) -> dict:
    """Per-draw issue slots, FP32 and SFU instructions of the timed kernel's executed common path, counted
    from the SASS of the library being timed (tools/sass_count.py); the last measured values if cuobjdump
    is unavailable."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import sass_count
        from paper_2005_10494_b200 import build
        return sass_count.pipe_mix(3, 0 if est == "cond" else 1, build.LIB)
    except Exception:
        return dict(PIPE_MIX_FALLBACK[est])


def issue_per_draw(est: str) -> float:
    return float(pipe_mix(est)["issue"])


ISSUE_LANES_PER_CLK_PER_SM = 128           # 4 SMSPs x 32 lanes, one warp-instruction per SMSP per clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--est", choices=["cond", "ind"], default="cond")
    ap.add_argument("--crn", action="store_true", help="NEXT f3: common random numbers per problem (not the headline)")
    ap.add_argument("--draws", type=int, default=W.DRAWS["C2"], help="draws per design per step (all ranks)")
    ap.add_argument("--problems", type=int, default=0, help="limit the C2 problem list (0 = all 513)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU work of the cpu_baseline sample")
    ap.add_argument("--no-tto-c2", action="store_true", help="skip the C2 time-to-optimal-design bookkeeping")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 dense-grid (strata prior) optimum")
    ap.add_argument("--no-n4", action="store_true", help="skip the n = 4 problem (N3 = 4000, d = 3 TPS)")
    ap.add_argument("--tto-draws", type=int, default=W.DRAWS["C3"],
                    help="draws/design of the time-to-optimal-design run (C3 slice); 0 = skip")
    return ap.parse_args()


# ----------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------------------------

def c2_specs(limit: int = 0):
    specs = W.c2_problems()
    return specs[:limit] if limit > 0 else specs


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2005_10494_b200 import mc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    est = mc.EST_COND if args.est == "cond" else mc.EST_IND
    specs = c2_specs(args.problems)
    t_prep0 = time.perf_counter()
    problems = [mc.problem_formula10(s.r, s.delta0(), s.i3, s.alpha0) for s in specs]
    alpha, pod = mc.candidates(problems, m=W.GRID_M, n3=W.N3, seed=W.SEED, device=local)
    t_cand = time.perf_counter() - t_prep0
    design = mc.Design(problems, alpha, pod, seed=W.SEED, estimator=est, device=local)
    if args.crn:
        design.set_sampling(True)
    # TPS plans before the MC pass (building them on a host thread during the first pass,
    # smooth_plan(wait=False), measured no faster: cuSOLVER's plan kernels and the fused kernel do not overlap)
    t1 = time.perf_counter()
    design.smooth_plan()
    torch.cuda.synchronize()
    t_plan = time.perf_counter() - t1
    D, N = design.D, int(args.draws)
    b, c = mc.shard_range(N, rank, world)
    stream = torch.cuda.current_stream()
    sums = design.new_sums()
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]

    def step(i=None):
        sums.zero_()
        if i is not None:
            kev[i][0].record(stream)
        design.evaluate(sums, b, c)
        if i is not None:
            kev[i][1].record(stream)
        mc.allreduce_sums(sums)
        mean, var = design.finalize(sums, N)
        sm, lam = design.smooth(mean, -1.0)
        idx, val, _ = design.argmax(sm, with_host=False)
        return idx, val, mean, var

    # warm-up step 1 doubles as the end of the C2 time-to-optimal-design run (BASELINE metric 2, the
    # secondary configuration): problem statement -> candidates -> plan -> one full pass -> the optimum
    # per problem (f1 L-BFGS on the TPS) -> the TPS over r and its maximum per scenario (f2).
    tto_c2 = None
    for wi in range(args.warmup):
        out_w = step()
        if wi == 0 and not args.no_tto_c2:
            _, _, mean_w, _ = out_w
            A_opt, v_opt, st_opt = design.refine(mean_w, -1.0)
            per_sc = {}
            for sc in ("a", "b", "c"):
                ks = [k for k, sp in enumerate(specs) if sp.scenario == sc and st_opt[k] != 1]
                if len(ks) < 4:
                    continue
                rr = np.array([specs[k].r[1:] for k in ks])
                surf = mc.Surface(rr, v_opt[ks], -1.0)
                r_star, p_star = surf.maximum()
                kbest = ks[int(np.argmax(v_opt[ks]))]
                per_sc[sc] = {"r_star": [float(x) for x in r_star], "power_r_star": float(p_star),
                              "best_lattice_r": [float(x) for x in specs[kbest].r[1:]],
                              "best_lattice_alpha": [float(x) for x in A_opt[kbest]],
                              "best_lattice_power": float(v_opt[kbest])}
            torch.cuda.synchronize()
            tt = torch.tensor([time.perf_counter() - t_prep0], dtype=torch.float64, device=f"cuda:{local}")
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tto_c2 = {"seconds": float(tt[0]), "workload": "C2: 513 problems x 2000 designs x 1e6 draws",
                      "includes": "candidates, thresholds, TPS plans, one MC pass, smoothing, per-problem L-BFGS "
                                  "optimum, TPS over r per scenario",
                      "per_scenario": per_sc,
                      "paper_printed": {"a": "0.6847 at r=(1,0,0)", "b": "0.783 (typo for 0.733, R15) at r2=0.365",
                                        "c": "0.977 at r=(1,0.446,0.168)"}}
    torch.cuda.synchronize()
    launches0 = design.launches
    clocks = Clocks(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        out = step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = design.launches - launches0
    ms = e0.elapsed_time(e1)
    kms = float(np.mean([a.elapsed_time(z) for a, z in kev]))
    t = torch.tensor([ms, kms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, kms = float(t[0]), float(t[1])
    draws_step = float(D) * N
    value = draws_step * args.steps / (ms * 1e-3)

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        alpha_pinned = torch.from_numpy(np.ascontiguousarray(alpha, dtype=np.float64)).pin_memory()
        res_idx = torch.empty(design.n_probs, dtype=torch.int64).pin_memory()
        res_val = torch.empty(design.n_probs, dtype=torch.float64).pin_memory()

        def e2e_step():
            design.upload(alpha_pinned)                       # H2D design table + device thresholds
            idx, val, _, _ = step()
            res_idx.copy_(idx, non_blocking=True)             # D2H per-problem optimum
            res_val.copy_(val, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return res_idx, res_val

        e2e_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        f1.record(stream)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1)
        te = torch.tensor([ems], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ems = float(te[0])
        e2e = {"value": draws_step * args.steps / (ems * 1e-3), "unit": "draws/s",
               "h2d_bytes_per_step": int(alpha_pinned.numel() * 8),
               "d2h_bytes_per_step": int(res_idx.numel() * 8 + res_val.numel() * 8),
               "ms_per_step": ems / args.steps}

    # ---- roofline of the dominant kernel (the fused MC kernel) ----
    draws_launch = float(D) * c
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    mhz = clk.get("sm_mhz") or 1965.0
    peak = ISSUE_LANES_PER_CLK_PER_SM * sm_count * (clk.get("sm_max_mhz") or 1965.0) * 1e6 / 1e12   # T lane-instr/s
    mix = pipe_mix(args.est)
    ipd = mix["issue"] if not args.crn else float("nan")
    achieved = ipd * draws_launch / (kms * 1e-3) / 1e12
    rate = draws_launch / (kms * 1e-3)
    fmax = (clk.get("sm_max_mhz") or 1965.0) * 1e6
    # the north star's "fraction of the FP32/SFU roofline": per-pipe achieved lane-op rates against the
    # pipe peaks (FP32 128 and MUFU 16 lane-ops/clk/SM, profiles/r01/pipes.json)
    pipes = None if args.crn else {
        "fp32": {"per_draw": mix["fp32"], "achieved": round(mix["fp32"] * rate / 1e12, 3),
                 "peak": round(128 * sm_count * fmax / 1e12, 3), "unit": "T lane-op/s",
                 "frac": round(mix["fp32"] * rate / (128 * sm_count * fmax), 4)},
        "sfu": {"per_draw": mix["sfu"], "achieved": round(mix["sfu"] * rate / 1e12, 3),
                "peak": round(16 * sm_count * fmax / 1e12, 3), "unit": "T lane-op/s",
                "frac": round(mix["sfu"] * rate / (16 * sm_count * fmax), 4)}}
    roof = {"bound": "alu", "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": "Tinst/s",
            "frac": round(achieved / peak, 4), "traffic": None,
            "traffic_ncu": {"dram_bytes_per_launch": 507904, "draws_per_launch": 1.2e10,
                            "capture": "profiles/r01/ncu_fused_cond_x2_summary.txt (--problems 6; the full C2 launch "
                                       "times out under --set full replay)",
                            "note": "DRAM bytes scale with designs (zc, problem_of_design, sums), not draws: "
                                    "~4e-5 B/draw; the kernel does no HBM work per draw"},
            "kernel": ("mc_crn_kernel" if args.crn else "mc_fused_kernel") + f"<3,{0 if est == 0 else 1},0>",
            "kernel_ms": round(kms, 3),
            "kernel_share_of_step": round(kms / (ms / args.steps), 4),
            "issue_per_draw": ipd,
            "pipes": pipes,
            "peak_basis": "128 lane-instr/clk/SM x SMs x sm_max_mhz (DESIGN.md §4)",
            "draws_per_s_kernel": draws_launch / (kms * 1e-3) * world}

    # the paper's own per-problem MC workload, literally (Formula 7 crossed, N1 = 10240, N2 = 20480 over
    # N3 = 2000 designs): one C2 problem through the crossed kernel (context, not the headline)
    paper_crossed = None
    if rank == 0 and not args.no_e2e:
        dx = mc.Design(problems[:1], alpha[pod == 0], np.zeros(int((pod == 0).sum()), dtype=np.int32), seed=W.SEED,
                       estimator=mc.EST_IND, device=local)
        sx = dx.new_sums()
        dx.evaluate_crossed(sx, 10240, 20480)
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        dx.evaluate_crossed(sx, 10240, 20480)
        c1.record(stream)
        torch.cuda.synchronize()
        cms = c0.elapsed_time(c1)
        paper_crossed = {"designs": int(dx.D), "N1": 10240, "N2": 20480, "ms": cms,
                         "pairs_per_s": dx.D * 10240 * 20480 / (cms * 1e-3),
                         "paper_reported_s_per_problem": 31.6,
                         "note": "paper: 4.5 h / 513 problems on a V100 incl. TPS and R/Python (P:343); context only"}
        dx.close()

    tto = None
    if args.tto_draws > 0:
        tto = time_to_optimal_design(args, mc, torch, dist, world, rank, local, est)
    c4 = None
    if not args.no_c4:
        c4 = c4_optimal_design(mc, torch, dist, world, rank, local, est)
    n4 = None
    if not args.no_n4:
        n4 = n4_optimal_design(mc, torch, dist, world, rank, local, est)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, specs, alpha, pod, seconds=args.cpu_seconds)

    if rank == 0:
        line = {"metric": "MC draws/sec (design x sample)", "value": value, "unit": "draws/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": "C2: paper 3-D problem (513 r-problems x 2000 alpha designs), 1e6 draws/design",
                           "problems": len(specs), "designs": D, "draws_per_design": N, "estimator": args.est,
                           "sampling": "common random numbers per problem" if args.crn else "independent per design",
                           "seed": W.SEED, "parallelism": f"sample-shard x{world} + int64 all_reduce",
                           "arithmetic": "f32 per-draw utility, exact int64 sums, f64 finalize and TPS",
                           "l2": "no flush: the per-step TPS plan read (~%.1f GB) exceeds L2" % (
                               8.0 * sum((pod == k).sum() ** 2 for k in range(len(specs))) / 1e9)},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "time_to_optimal_design": tto, "time_to_optimal_design_c2": tto_c2,
                "c4_optimal_design": c4, "n4_optimal_design": n4,
                "paper_literal_crossed_problem": paper_crossed,
                "clocks": clk,
                "prep_s": {"candidates": round(t_cand, 3), "tps_plan": round(t_plan, 3)},
                "best_design_first_problem": int(out[0][0].item())}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def time_to_optimal_design(args, mc, torch, dist, world, rank, local, est):
    """BASELINE metric 2: wall-clock from the problem statement to the optimal design on the host,
    for the C3 headline slice (scenario (c), r = (1, .45, .15), every valid m = 64 alpha design) at
    `tto_draws` draws per design sharded over the ranks: candidates (GPU alpha_n solve) -> design
    init -> TPS plan -> fused MC -> all_reduce -> finalize -> TPS+GCV -> argmax -> host."""
    spec = W.c2_slice()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = mc.problem_formula10(spec.r, spec.delta0(), spec.i3, spec.alpha0)
    alpha, pod = mc.candidates([prob], m=W.GRID_M, n3=0, seed=W.SEED, device=local)
    dsg = mc.Design([prob], alpha, pod, seed=W.SEED, estimator=est, device=local)
    dsg.smooth_plan(wait=False)      # overlaps the MC pass; evaluate_design_objective's smooth() joins it
    res = mc.evaluate_design_objective(dsg, args.tto_draws, lam=-1.0, rank=rank, world=world)
    best, val = res.best
    t1 = time.perf_counter()
    tt = torch.tensor([t1 - t0], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    raw = res.mean.cpu().numpy()
    se = np.sqrt(res.var.cpu().numpy() / args.tto_draws)
    out = {"seconds": float(tt[0]), "workload": "C3 slice: scenario (c), r=(1,0.45,0.15), all valid m=64 designs",
           "designs": int(dsg.D), "draws_per_design": int(args.tto_draws), "n_gpus": world,
           "best_design": int(best), "best_alpha": [float(x) for x in alpha[best]], "P_smoothed": float(val),
           "P_hat": float(raw[best]), "SE": float(se[best]), "raw_argmax": int(np.argmax(raw)),
           "lambda": float(res.lam_used.cpu().numpy()[0])}
    dsg.close()
    return out


def n4_optimal_design(mc, torch, dist, world, rank, local, est):
    """The paper's n = 4 workload (N3 = 4000 designs, a 3-D TPS): one problem from the statement to
    the continuous optimum — candidates (m = 32 grid over alpha_1..3, alpha_4 solved on the GPU, seeded
    N3 subset) -> MC (1e6 draws/design) -> all_reduce -> finalize -> TPS plan (N = 4000) + GCV -> argmax
    -> L-BFGS on the 3-D TPS (f1)."""
    spec = W.n4_problem()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = mc.problem_formula10(spec.r, spec.delta0(), spec.i3, spec.alpha0)
    alpha, pod = mc.candidates([prob], m=W.N4_GRID_M, n3=W.N4_N3, seed=W.SEED, device=local)
    dsg = mc.Design([prob], alpha, pod, seed=W.SEED, estimator=est, device=local)
    res = mc.evaluate_design_objective(dsg, W.DRAWS["C2"], lam=-1.0, rank=rank, world=world)
    best, val = res.best
    A, v, st = dsg.refine(res.mean, -1.0)
    t1 = time.perf_counter()
    tt = torch.tensor([t1 - t0], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    out = {"seconds": float(tt[0]), "workload": "n = 4, r = (1, 0.6, 0.35, 0.15), scenario (c), N3 = 4000 of the "
           "m = 32 grid, 1e6 draws/design", "designs": int(dsg.D), "best_design": int(best),
           "best_alpha": [float(x) for x in alpha[best]], "P_smoothed": float(val),
           "alpha_opt": [float(x) for x in A[0]], "P_opt": float(v[0]), "refine_status": int(st[0]),
           "lambda": float(res.lam_used.cpu().numpy()[0])}
    dsg.close()
    return out


def c4_optimal_design(mc, torch, dist, world, rank, local, est):
    """Configuration C4 (BASELINE configs[3]; synthetic strata prior): 256 cutoffs r2 x 256 alpha_1 designs
    (alpha_2 solved) x 1e6 draws, wall-clock from the problem statement to the optimal (r2, alpha) on the
    host: candidates -> fused MC (strata prior) -> all_reduce -> finalize -> separable kernel smoother
    with GCV -> argmax."""
    from paper_2005_10494_b200 import sweep
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = sweep.c4_grid_optimum(W.c4_r2_values(), 211.0, W.C4_STRATA, W.C4_GRID, W.DRAWS["C4"], W.SEED, est=est,
                              device=local, rank=rank, world=world)
    t1 = time.perf_counter()
    tt = torch.tensor([t1 - t0], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return {"seconds": float(tt[0]), "workload": "C4: 256 r2 x 256 alpha_1 designs (alpha_2 solved), 5-D strata prior, "
            "1e6 draws/design", "designs": int(g.mean.size), "draws_per_design": W.DRAWS["C4"], "n_gpus": world,
            "r2_star": g.r2, "alpha_star": [float(x) for x in g.alpha], "P_smoothed": g.power_smoothed,
            "P_hat": g.power_hat, "SE": g.se, "bandwidths": [float(x) for x in g.bandwidths],
            "P_hat_range": [float(g.mean.min()), float(g.mean.max())],
            "survey_anchor": "SURVEY A.11: max ~0.941 at r2=0.3, alpha_1 ~0.002-0.008; range 0.797-0.941 (coarse 4e5-draw MC)"}


# ----------------------------------------------------------------------------------------------
# CPU oracle (cpu_baseline and --impl reference).  The ONLY places bench.py executes oracle/.

def _oracle_worker(job):
    from oracle import oracle as O
    r, delta0, i3, alpha0, a, est, seed, design, N = job
    prob = O.formula10_problem(r, delta0, i3, alpha0)
    t = time.perf_counter()
    s = O.design_sums(prob, a, est, seed, design, 0, N)
    return s.tolist(), time.perf_counter() - t


def _oracle_jobs(specs, alpha, pod, designs, est, N):
    jobs = []
    for d in designs:
        s = specs[int(pod[d])]
        jobs.append((s.r, s.delta0(), s.i3, s.alpha0, alpha[d].tolist(), est, W.SEED, int(d), N))
    return jobs


def cpu_baseline(args, specs, alpha, pod, seconds=12.0):
    """The oracle as it stands (single-threaded C, fp64), one process per host core, on a bounded
    sample of the same workload: evenly spaced designs of the C2 list at the full 1e6 draws each."""
    import multiprocessing as mp
    from oracle import oracle as O
    O.build()
    cores = os.cpu_count() or 1
    est = 0 if args.est == "cond" else 1
    rate_guess = 1.2e6 if est == 0 else 1.7e6
    N = int(args.draws)
    n_des = max(cores, int(seconds * rate_guess * cores / N))
    designs = np.linspace(0, len(alpha) - 1, n_des).astype(np.int64)
    jobs = _oracle_jobs(specs, alpha, pod, designs, est, N)
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_oracle_worker, jobs, chunksize=1)
    wall = time.perf_counter() - t0
    draws = float(N) * len(jobs)
    return {"value": draws / wall, "unit": "draws/s", "cores": cores, "kind": "oracle",
            "sample": f"{len(jobs)} evenly spaced C2 designs x {N} draws (est={args.est}), "
                      f"{cores} single-threaded oracle processes, wall {wall:.1f} s",
            "per_core": draws / sum(r[1] for r in res)}


def run_reference(args):
    """--impl reference: the oracle (the reference arm for this tier) on the box's host cores, on
    this arm's config/metric; rank 0 only under torchrun."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import multiprocessing as mp
    from oracle import oracle as O
    O.build()
    specs = c2_specs(args.problems)
    cores = os.cpu_count() or 1
    est = 0 if args.est == "cond" else 1
    N = int(args.draws)
    # bounded sample per step: `cores` designs (one per core) of the C2 workload, each a random
    # oracle-solved alpha grid point of an evenly spaced problem, at the full draws per design
    rng = np.random.default_rng(W.SEED & 0xFFFF)
    n_des = cores
    probs_idx = np.linspace(0, len(specs) - 1, n_des).astype(int)
    alpha, pod = [], []
    for k in probs_idx:
        s = specs[k]
        while True:
            a1, a2 = (rng.integers(0, W.GRID_M, 2) + 0.5) * s.alpha0 / W.GRID_M
            a3 = O.solve_alpha_n(s.r, s.alpha0, [a1, a2], 1e-12)
            if a3 is not None:
                break
        alpha.append([a1, a2, a3])
        pod.append(k)
    alpha, pod = np.array(alpha), np.array(pod)
    jobs = _oracle_jobs(specs, alpha, pod, np.arange(n_des), est, N)

    def one_step(pool):
        res = pool.map(_oracle_worker, jobs, chunksize=1)
        sums = np.array([r[0] for r in res], dtype=np.int64)
        mean, var = O.finalize(sums, N)
        return O.argmax(mean)

    with mp.get_context("fork").Pool(cores) as pool:
        for _ in range(args.warmup):
            one_step(pool)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            one_step(pool)
        wall = time.perf_counter() - t0
    draws = float(N) * n_des * args.steps
    value = draws / wall
    line = {"impl": "reference", "metric": "MC draws/sec (design x sample)", "value": value, "unit": "draws/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2: paper 3-D problem (513 r-problems x 2000 alpha designs), 1e6 draws/design",
                       "estimator": args.est, "draws_per_design": N},
            "cpu_baseline": {"value": value, "unit": "draws/s", "cores": cores, "kind": "oracle",
                             "sample": f"per step {n_des} C2 designs (one per core) x {N} draws, oracle fp64 C"},
            "e2e": {"value": value, "unit": "draws/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
