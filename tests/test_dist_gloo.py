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
