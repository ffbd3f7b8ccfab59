"""Edge and degenerate cases of the CUDA path (empty / ragged inputs, alpha = 0, n = 1, limits, errors)."""
import math

import numpy as np
import pytest

from paper_2005_10494_b200 import workloads as W
from tests.helpers import lib_problem, oracle_problem

pytestmark = pytest.mark.gpu
SEED = W.SEED


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def mc(torch):
    from paper_2005_10494_b200 import build, mc as m
    build.build()
    return m


@pytest.mark.parametrize("est", [0, 1])
@pytest.mark.parametrize("crn", [False, True])
def test_alpha_zero_never_rejects(O, mc, torch, est, crn):
    spec = W.c2_slice()
    alpha = np.array([[0.0, 0.0, 0.0], [0.0, 0.0, 0.025], [0.0025, 0.0138, 0.0128]])
    dsg = mc.Design([lib_problem(mc, spec)], alpha, np.zeros(3, dtype=np.int32), seed=SEED, estimator=est)
    dsg.set_sampling(crn)
    s = dsg.new_sums()
    dsg.evaluate(s, 0, 10_000)
    S = s.cpu().numpy()
    assert S[0, 0] == 0 and S[0, 1] == 0                       # z = +inf everywhere: u = 0 exactly
    op = oracle_problem(O, spec)
    ref = O.design_sums(op, alpha[1], est, SEED, 0 if crn else 1, 0, 10_000, tag=1 if crn else 0)
    if est == 0:
        assert abs(S[1, 0] - ref[0]) <= 1e-5 * ref[0]
    else:
        assert abs(int(S[1, 0]) - int(ref[0])) <= 2 * 2**23


def test_empty_and_single_sample_calls(O, mc, torch):
    spec = W.c2_slice()
    alpha = np.array([[0.0025, 0.0138, 0.0128], [0.01, 0.005, 0.0123]])
    dsg = mc.Design([lib_problem(mc, spec)], alpha, np.zeros(2, dtype=np.int32), seed=SEED)
    s = dsg.new_sums()
    dsg.evaluate(s, 0, 0)                       # no samples: no-op
    dsg.evaluate(s, 5, 10, design_begin=1, design_count=0)
    assert int(s.abs().sum()) == 0
    dsg.evaluate(s, 12_345, 1)                  # one sample, odd position in its Philox step
    op = oracle_problem(O, spec)
    for d in range(2):
        ref = O.design_sums(op, alpha[d], 0, SEED, d, 12_345, 1)
        assert abs(int(s[d, 0]) - int(ref[0])) <= 200        # one draw: |du| <= 5e-5 -> < 420 units of 2^-23
    with pytest.raises(mc.McError):
        dsg.evaluate(s, 2**40, 1)               # beyond the int64 headroom of 2^40 draws per design
    with pytest.raises(mc.McError):
        dsg.evaluate(s, 2**40 - 1, 1)           # exactly 2^40 sample indices: 2^40 x 2^23 = 2^63 overflows
    dsg.evaluate(s, 2**40 - 2, 1)               # the last admissible sample index
    with pytest.raises(mc.McError):
        dsg.evaluate(s, 0, 10, design_begin=1, design_count=5)
    with pytest.raises(mc.McError):
        dsg.set_launch(48, 0)                   # not a multiple of 32
    with pytest.raises(mc.McError):
        dsg.finalize(s, 0)


def test_n1_problems_batch_smooth_and_argmax(O, mc, torch):
    """n = 1 (the paper's scenario (a) optimum has no subsets): COND is exact per draw for a point mass;
    smoothing passes through; argmax per problem."""
    probs = [mc.problem_formula10([1.0], [d0], 127.0) for d0 in (0.2, 0.25, 0.3)]
    alpha = np.array([[0.025], [0.025], [0.025], [0.02]])
    pod = np.array([0, 1, 2, 2], dtype=np.int32)
    dsg = mc.Design(probs, alpha, pod, seed=SEED)
    res = mc.evaluate_design_objective(dsg, 50_000)
    m = res.mean.cpu().numpy()
    assert np.allclose(res.smoothed.cpu().numpy(), m)
    assert m[0] < m[1] < m[2]
    assert res.idx.cpu().numpy().tolist() == [0, 1, 2 if m[2] >= m[3] else 3]
    for d, (p, a) in enumerate(zip([0.2, 0.25, 0.3, 0.3], alpha)):
        exact = O.assurance_gaussian(O.formula10_problem([1.0], [p], 127.0), a)
        v = res.var.cpu().numpy()[d]
        assert abs(m[d] - exact) < 5 * math.sqrt(v / 50_000)


def test_design_upload_roundtrip(O, mc, torch):
    spec = W.c2_slice()
    a1 = np.array([[0.0025, 0.0138, 0.0128], [0.01, 0.005, 0.0123]])
    a2 = np.array([[0.01, 0.005, 0.0123], [0.0025, 0.0138, 0.0128]])
    dsg = mc.Design([lib_problem(mc, spec)], a1, np.zeros(2, dtype=np.int32), seed=SEED)
    s1 = dsg.new_sums()
    dsg.evaluate(s1, 0, 20_000)
    dsg.upload(torch.from_numpy(a2).pin_memory())
    s2 = dsg.new_sums()
    dsg.evaluate(s2, 0, 20_000)
    d2 = mc.Design([lib_problem(mc, spec)], a2, np.zeros(2, dtype=np.int32), seed=SEED)
    s3 = d2.new_sums()
    d2.evaluate(s3, 0, 20_000)
    assert torch.equal(s2, s3) and not torch.equal(s1, s2)
    with pytest.raises(mc.McError):
        dsg.upload(np.array([[0.03, 0.0, 0.0], [0.0, 0.0, 0.0]]))


def test_c2_full_size_sampled_parity(O, mc, torch):
    """BASELINE configs[1] at full size in the bench's launch configuration: 513 problems x 2000 designs
    x 1e6 draws on the GPU; 6 sampled designs recomputed by the oracle (which re-solves alpha_3 from the
    design's grid coordinates itself) within 1e-5 relative."""
    specs = W.c2_problems()
    probs = [lib_problem(mc, s) for s in specs]
    alpha, pod = mc.candidates(probs, m=W.GRID_M, n3=W.N3, seed=W.SEED)
    assert alpha.shape == (513 * 2000, 3)
    dsg = mc.Design(probs, alpha, pod, seed=SEED)
    N = 1_000_000
    s = dsg.new_sums()
    dsg.evaluate(s, 0, N)
    mean = dsg.finalize(s, N)[0].cpu().numpy()
    rng = np.random.default_rng(5)
    for d in rng.choice(len(alpha), 6, replace=False):
        sp = specs[pod[d]]
        a12 = alpha[d, :2]
        k = np.round(a12 / sp.alpha0 * W.GRID_M - 0.5)
        assert np.allclose((k + 0.5) * sp.alpha0 / W.GRID_M, a12, rtol=0, atol=1e-18)   # a grid point
        a3 = O.solve_alpha_n(sp.r, sp.alpha0, a12, 1e-14)
        assert a3 is not None and abs(a3 - alpha[d, 2]) < 1e-11
        ref = O.finalize(O.design_sums(oracle_problem(O, sp), [a12[0], a12[1], a3], 0, SEED, int(d), 0, N), N)[0][0]
        assert abs(mean[d] - ref) <= 1e-5 * ref, (d, mean[d], ref)


def test_checkpoint_resume_is_bit_identical(O, mc, torch, tmp_path):
    spec = W.c2_slice()
    alpha = np.array([[0.0025, 0.0138, 0.0128], [0.01, 0.005, 0.0123]])
    dsg = mc.Design([lib_problem(mc, spec)], alpha, np.zeros(2, dtype=np.int32), seed=SEED)
    full = dsg.new_sums()
    dsg.evaluate(full, 0, 300_001)
    part = dsg.new_sums()
    dsg.evaluate(part, 0, 123_457)
    mc.checkpoint_save(str(tmp_path / "ck"), part, 123_457, SEED)
    s, done, seed, _ = mc.checkpoint_load(str(tmp_path / "ck"))
    resumed = torch.from_numpy(s).cuda()
    dsg.evaluate(resumed, done, 300_001 - done)
    assert seed == SEED and torch.equal(resumed, full)


def test_sums_buffer_is_validated(mc, torch):
    """The 64-bit atomics write sums[2d], sums[2d+1]: any buffer other than a contiguous int64 (D, 2) CUDA
    tensor on the ctx device is rejected before a kernel runs."""
    spec = W.c2_slice()
    alpha = np.array([[0.0025, 0.0138, 0.0128], [0.01, 0.005, 0.0123]])
    dsg = mc.Design([lib_problem(mc, spec)], alpha, np.zeros(2, dtype=np.int32), seed=SEED)
    bad = [torch.zeros((2, 2), dtype=torch.int32, device="cuda"),          # int32: atomics would overrun
           torch.zeros((2, 4), dtype=torch.int64, device="cuda")[:, ::2],  # non-contiguous view
           torch.zeros((4,), dtype=torch.int64, device="cuda"),            # right numel, wrong shape
           torch.zeros((2, 2), dtype=torch.int64)]                         # host tensor
    for s in bad:
        with pytest.raises(ValueError):
            dsg.evaluate(s, 0, 10)
        with pytest.raises(ValueError):
            dsg.finalize(s, 10)
    dsg.close()


def test_crossed_rejects_int64_overflow(mc, torch):
    """S2 = sum_k c_k^2 <= N1 N2^2 must fit int64: N1 N2^2 >= 2^63 is rejected up front."""
    spec = W.c2_slice()
    dsg = mc.Design([lib_problem(mc, spec)], np.array([[0.0025, 0.0138, 0.0128]]), np.zeros(1, dtype=np.int32),
                    seed=SEED, estimator=mc.EST_IND)
    s = dsg.new_sums()
    with pytest.raises(mc.McError):
        dsg.evaluate_crossed(s, 2**31, 2**16)          # exactly 2^63
    dsg.evaluate_crossed(s, 1000, 2**16)               # fine
    assert int(s[0, 0]) > 0
    dsg.close()


@pytest.mark.parametrize("est", [0, 1])
def test_alpha_zero_never_rejects_n10(O, mc, torch, est):
    """Reading R25: the kernel's normal CDF holds q at 2.0e-9 beyond x = 5.887; ten such stages stay below
    half a 2^-23 step, so the all-zero design (z = +inf everywhere) has u = 0 exactly at n = 10 too."""
    spec = W.c5_problem(10)
    dsg = mc.Design([lib_problem(mc, spec)], np.zeros((1, 10)), np.zeros(1, dtype=np.int32), seed=SEED, estimator=est)
    s = dsg.new_sums()
    dsg.evaluate(s, 0, 200_000)
    assert int(s[0, 0]) == 0 and int(s[0, 1]) == 0
    dsg.close()
