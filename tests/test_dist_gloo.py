"""Multi-GPU host logic on CPU (world_size 2, gloo): the rank sample shards of mc.shard_range and the
single int64 SUM all_reduce (row a7) reproduce the single-rank sums bit-for-bit.  The per-rank sums
are computed by the oracle (the CUDA kernel needs a GPU; its shard invariance is tested in
tests/test_gpu_parity.py::test_sums_invariant_to_launch_shape_and_splits)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2005_10494_b200 import mc
    from paper_2005_10494_b200 import workloads as W
    spec = W.c2_slice()
    prob = O.formula10_problem(spec.r, spec.delta0(), spec.i3, spec.alpha0)
    alpha = [[0.002, 0.0138, 0.0128], [0.01, 0.005, 0.0123]]
    N = 6_001
    b, c = mc.shard_range(N, rank, world)
    sums = torch.zeros((len(alpha), 2), dtype=torch.int64)
    for d, a in enumerate(alpha):
        sums[d] = torch.from_numpy(O.design_sums(prob, a, 0, W.SEED, d, b, c))
    mc.allreduce_sums(sums)
    if rank == 0:
        q.put(sums.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_allreduce_equals_single_rank(O, world):
    from paper_2005_10494_b200 import workloads as W
    ctx = tmp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = 29500 + world + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    spec = W.c2_slice()
    prob = O.formula10_problem(spec.r, spec.delta0(), spec.i3, spec.alpha0)
    ref = np.stack([O.design_sums(prob, a, 0, W.SEED, d, 0, 6_001)
                    for d, a in enumerate([[0.002, 0.0138, 0.0128], [0.01, 0.005, 0.0123]])])
    assert np.array_equal(got, ref)


def _gpu_worker(rank, world, port, q):
    """One rank of the multi-GPU path on a single device: this rank's Philox sample shard through the CUDA
    kernel (mc_evaluate_grid), the sums copied to the host, the single int64 SUM all_reduce over gloo
    (row a7; NCCL in bench.py), then finalize on the device."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2005_10494_b200 import mc
    from paper_2005_10494_b200 import workloads as W
    torch.cuda.set_device(0)
    spec = W.c2_slice()
    prob = mc.problem_formula10(spec.r, spec.delta0(), spec.i3, spec.alpha0)
    alpha = np.array([[0.002, 0.0138, 0.0128], [0.01, 0.005, 0.0123], [0.0, 0.0, 0.025]])
    for est in (mc.EST_COND, mc.EST_IND):
        dsg = mc.Design([prob], alpha, np.zeros(len(alpha), dtype=np.int32), seed=W.SEED, estimator=est)
        N = 1_000_003
        b, c = mc.shard_range(N, rank, world)
        sums = dsg.new_sums()
        dsg.evaluate(sums, b, c)
        host = sums.cpu()
        mc.allreduce_sums(host)
        mean, _ = dsg.finalize(host.cuda(), N)
        if rank == 0:
            q.put((est, host.numpy().copy(), mean.cpu().numpy().copy()))
        dsg.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_gpu_shards_allreduce_equal_single_rank(world):
    """CUDA-produced per-rank sums through the collective.  `world` gloo ranks share one GPU
    (no kernel waits on another rank); their all_reduced int64 sums equal one rank's full-range sums bit for
    bit, for both estimators."""
    from paper_2005_10494_b200 import mc
    from paper_2005_10494_b200 import workloads as W
    ctx = tmp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = 29600 + world + (os.getpid() % 1000)
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get() for _ in range(2)]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    spec = W.c2_slice()
    prob = mc.problem_formula10(spec.r, spec.delta0(), spec.i3, spec.alpha0)
    alpha = np.array([[0.002, 0.0138, 0.0128], [0.01, 0.005, 0.0123], [0.0, 0.0, 0.025]])
    for est, sums, mean in got:
        dsg = mc.Design([prob], alpha, np.zeros(len(alpha), dtype=np.int32), seed=W.SEED, estimator=est)
        ref = dsg.new_sums()
        dsg.evaluate(ref, 0, 1_000_003)
        assert np.array_equal(sums, ref.cpu().numpy()), est
        assert np.array_equal(mean, dsg.finalize(ref, 1_000_003)[0].cpu().numpy())
        dsg.close()


def _smooth_worker(rank, world, port, q):
    """One rank of the sharded smoothing: plans and smooths the problems k with k mod world == rank, runs
    L-BFGS on them, and the all_reduce assembles every problem's results on all ranks."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dsg, mean = _smooth_setup()
    dsg.smooth_plan_sharded(rank, world)
    sm, lam = dsg.smooth_sharded(mean, -1.0, rank, world)
    A, v, st = dsg.refine_sharded(mean, -1.0, rank, world)
    if rank == 0:
        q.put((sm.cpu().numpy(), lam.cpu().numpy(), A, v, st))
    dsg.close()
    dist.barrier()
    dist.destroy_process_group()


def _smooth_setup():
    from paper_2005_10494_b200 import mc
    from paper_2005_10494_b200 import workloads as W
    specs = W.c2_problems()[::60][:7]
    probs = [mc.problem_formula10(s.r, s.delta0(), s.i3, s.alpha0) for s in specs]
    alpha, pod = mc.candidates(probs, m=16, n3=100, seed=W.SEED)
    dsg = mc.Design(probs, alpha, pod, seed=W.SEED)
    sums = dsg.new_sums()
    dsg.evaluate(sums, 0, 200_000)
    mean, _ = dsg.finalize(sums, 200_000)
    return dsg, mean


@pytest.mark.gpu
def test_sharded_smoothing_equals_single_rank():
    """Multi-GPU smoothing: 3 gloo ranks on one GPU each plan / smooth / refine the problems
    they own; the assembled smoothed values, lambdas and continuous optima equal one rank's (batched
    eigensolves of different batch compositions: values within 1e-12, the maximisers within 1e-7)."""
    ctx = tmp.get_context("spawn")
    q = ctx.SimpleQueue()
    world = 3
    port = 29700 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_smooth_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    sm, lam, A, v, st = q.get()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    dsg, mean = _smooth_setup()
    rs, rl = dsg.smooth(mean, -1.0)
    rA, rv, rst = dsg.refine(mean, -1.0)
    dsg.close()
    assert np.array_equal(lam, rl.cpu().numpy())
    assert np.allclose(sm, rs.cpu().numpy(), rtol=0, atol=1e-12)
    assert np.array_equal(st, rst)
    assert np.allclose(v, rv, rtol=0, atol=1e-12)
    # the maximiser of a flat maximum moves ~sqrt(1e-13) with 1e-13 changes of the spline: alpha within 1e-7
    assert np.allclose(A, rA, rtol=0, atol=1e-7)


def _nccl_worker(port, q):
    """World size 1 over NCCL on the box's one GPU: the device-resident int64 sums the kernel wrote go through
    NCCL's SUM all_reduce in place (the exchange bench.py runs at N > 1; mc.allreduce_sums is the identity at
    world 1, so the collective is called directly here)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    from paper_2005_10494_b200 import mc
    from paper_2005_10494_b200 import workloads as W
    spec = W.c2_slice()
    prob = mc.problem_formula10(spec.r, spec.delta0(), spec.i3, spec.alpha0)
    alpha = np.array([[0.002, 0.0138, 0.0128], [0.01, 0.005, 0.0123], [0.0, 0.0, 0.025]])
    dsg = mc.Design([prob], alpha, np.zeros(len(alpha), dtype=np.int32), seed=W.SEED)
    sums = dsg.new_sums()
    dsg.evaluate(sums, 0, 1_000_003)
    before = sums.cpu().numpy().copy()
    dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    torch.cuda.synchronize()
    q.put((dist.get_backend(), before, sums.cpu().numpy().copy()))
    dsg.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_allreduce_of_kernel_sums_world1():
    """Row a7 over NCCL: the pool gives one GPU per box, so NCCL runs at world size 1 — the
    CUDA-produced device sums pass through an NCCL int64 SUM all_reduce unchanged.  The multi-rank exchange
    itself is covered by the gloo tests above."""
    ctx = tmp.get_context("spawn")
    q = ctx.SimpleQueue()
    p = ctx.Process(target=_nccl_worker, args=(29800 + (os.getpid() % 1000), q))
    p.start()
    backend, before, after = q.get()
    p.join(timeout=300)
    assert p.exitcode == 0
    assert backend == "nccl"
    assert before[:, 0].min() > 0 and np.array_equal(before, after)
