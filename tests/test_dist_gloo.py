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
