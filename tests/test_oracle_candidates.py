"""Pins for the oracle's alpha grid, alpha_n solve and N3 subset (Sec. 2.1, 2.3; Formula 2)."""
import numpy as np
import pytest


def test_alpha_n_roundtrip_and_n1(O):
    assert O.solve_alpha_n([1.0], 0.025, []) == 0.025        # S:256 single test uses the budget
    r = [1, 0.5]
    a2 = O.solve_alpha_n(r, 0.025, [0.02])
    assert O.fwer(r, [0.02, a2]) == pytest.approx(0.025, abs=1e-12)
    assert a2 == pytest.approx(0.0086893, abs=1e-6)            # S:262 (cross-check)
    # second test disabled leaves the exact budget: alpha_2 = 0
    assert O.solve_alpha_n(r, 0.025, [0.025]) == 0.0
    r3 = [1, 0.45, 0.15]
    a3 = O.solve_alpha_n(r3, 0.025, [0.004, 0.012])
    assert O.fwer(r3, [0.004, 0.012, a3]) == pytest.approx(0.025, abs=1e-12)


def test_infeasible_points_are_dropped(O):
    # FWER(0.0225, 0.0225, 0) already exceeds alpha0 for r=(1,.5,.25): infeasible (S:275 note)
    assert O.fwer([1, 0.5, 0.25], [0.0225, 0.0225, 0.0]) > 0.025
    assert O.solve_alpha_n([1, 0.5, 0.25], 0.025, [0.0225, 0.0225]) is None


def test_alpha_sum_exceeds_alpha0(O):
    # correlated nested tests allow alpha_1 + alpha_2 + alpha_3 > alpha0.
    r = [1, 0.5, 0.25]
    a3 = O.solve_alpha_n(r, 0.025, [0.012, 0.012])
    assert a3 is not None and 0.012 + 0.012 + a3 > 0.025


def test_grid_n2_layout(O):
    r = [1, 0.3]
    A, ok = O.alpha_grid(r, 0.025, 16)
    assert A.shape == (16, 2)
    assert np.allclose(A[:, 0], (np.arange(16) + 0.5) * 0.025 / 16)
    assert ok.all()      # for n = 2 every alpha_1 < alpha0 leaves room for alpha_2
    for a in A:
        assert O.fwer(r, a) == pytest.approx(0.025, abs=1e-12)
        assert 0 <= a[1] <= 0.025


def test_grid_n3_small(O):
    r = [1, 0.45, 0.15]
    m = 8
    A, ok = O.alpha_grid(r, 0.025, m)
    assert A.shape == (m * m, 3)
    # first free coordinate slowest
    assert np.allclose(A[:, 0], np.repeat((np.arange(m) + 0.5) * 0.025 / m, m))
    assert np.allclose(A[:, 1], np.tile((np.arange(m) + 0.5) * 0.025 / m, m))
    for a, v in zip(A, ok):
        f0 = O.fwer(r, [a[0], a[1], 0.0])
        assert v == (f0 <= 0.025)
        if v:
            assert O.fwer(r, a) == pytest.approx(0.025, abs=1e-12)


def test_subset_properties(O):
    s = O.subset(2495, 2000, 0x2005105494)
    assert len(s) == 2000 and len(set(s.tolist())) == 2000
    assert np.all(np.diff(s) > 0) and s[0] >= 0 and s[-1] < 2495
    assert np.array_equal(s, O.subset(2495, 2000, 0x2005105494))
    assert not np.array_equal(s, O.subset(2495, 2000, 0x2005105495))
    # n3 = V selects everything
    assert np.array_equal(O.subset(50, 50, 1), np.arange(50))
    # roughly uniform inclusion: each of 10 bins of 100 gets ~ 50 of 500
    t = O.subset(1000, 500, 3)
    cnt = np.bincount(t // 100, minlength=10)
    assert cnt.min() > 25 and cnt.max() < 75


def test_r_lattice_count():
    # 171 valid pairs 1 > r2 > r3 > 0 on the step-0.05 lattice
    from paper_2005_10494_b200 import workloads
    pairs = workloads.r_lattice(0.05)
    assert len(pairs) == 171
    assert all(1 > a > b > 0 for a, b in pairs)
