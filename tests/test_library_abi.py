"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/*.h declares, and its
host-only helpers (thresholds, Eq. 9, Formula 10, validation) behave.  No compute calls."""
import ctypes
import glob
import math
import os
import re

import numpy as np
import pytest
from scipy import special

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mc():
    from paper_2005_10494_b200 import build, mc as m
    build.build()
    return m


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for mt in re.finditer(r"\b(mc_[a-z0-9_]+)\s*\(", src):
            names.add(mt.group(1))
    return names


def test_exports_every_declared_symbol(mc):
    L = mc.lib()
    names = _declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name
    assert set(mc.EXPORTED) == names


def test_library_is_sm100a_only(mc):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {mc.lib_path()}").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(7|8|9)\d", out)


def test_threshold_fp64(mc):
    for a in np.concatenate([np.logspace(-14, -0.31, 200), [0.025, 0.0125]]):
        assert mc.threshold(a) == pytest.approx(-special.ndtri(a), rel=2e-15)
    assert math.isinf(mc.threshold(0.0))
    assert math.isnan(mc.threshold(-0.1)) and math.isnan(mc.threshold(1.0))


def test_information_units_eq9(mc):
    assert round(mc.information_units(0.025, 0.1, 0.25)) == 127
    assert round(mc.information_units(0.025, 0.1, 0.20)) == 211
    assert math.isnan(mc.information_units(0.025, 0.1, 1.5))


def test_formula10_problem(mc):
    r = [1.0, 0.5]
    p = mc.problem_formula10(r, [0.2, 0.25], 211.0)
    assert p.theta[0] == pytest.approx(0.223144, abs=1e-6) and p.theta[1] == pytest.approx(0.287682, abs=1e-6)
    assert p.sigma[0] == pytest.approx(1 / math.sqrt(20)) and p.sigma[1] == pytest.approx(2 * 0.2236068 / math.sqrt(2), rel=1e-6)
    with pytest.raises(mc.McError) as e:
        mc.problem_formula10([1.0, 1.2], [0.2, 0.2], 211.0)
    assert e.value.status == 1 and "decreasing" in str(e.value)
    with pytest.raises(mc.McError):
        mc.problem_formula10([1.0, 0.5], [0.2, 1.5], 211.0)


@pytest.mark.parametrize("bad", ["r0", "ratio", "alpha0", "i3", "alpha_range", "pod_order"])
def test_design_init_validation_before_device(mc, bad):
    # every validation happens on the host before any CUDA call, so these run without a GPU
    r = [1.0, 0.45, 0.15]
    p = mc.problem_formula10(r, [0.2, 0.53, 0.71], 211.0)
    alpha = np.array([[0.002, 0.0138, 0.0128], [0.003, 0.01, 0.012]])
    pod = np.array([0, 0], dtype=np.int32)
    if bad == "r0":
        p.r[0] = 0.9
    elif bad == "ratio":
        p.r[2] = p.r[1] * (1 - 1e-8)
    elif bad == "alpha0":
        p.alpha0 = 0.7
    elif bad == "i3":
        p.i3 = -1.0
    elif bad == "alpha_range":
        alpha[1, 2] = 0.03
    elif bad == "pod_order":
        p2 = mc.problem_formula10(r, [0.2, 0.53, 0.71], 211.0)
        arr = (mc.mc_problem * 2)(p, p2)
        pod = np.array([1, 0], dtype=np.int32)
        ctx = ctypes.c_void_p()
        st = mc.lib().mc_design_init(ctypes.byref(ctx), arr, 2, alpha.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                     pod.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), 2, 1, 0, 0)
        assert st == 1 and b"non-decreasing" in mc.lib().mc_last_error()
        return
    arr = (mc.mc_problem * 1)(p)
    ctx = ctypes.c_void_p()
    st = mc.lib().mc_design_init(ctypes.byref(ctx), arr, 1, alpha.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                 pod.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), 2, 1, 0, 0)
    assert st == 1, mc.lib().mc_last_error()


def test_compute_calls_refuse_without_cuda(mc, monkeypatch):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mc.Design([mc.problem_formula10([1.0], [0.25], 127.0)], [[0.025]], [0], seed=1)


def test_shard_range_partitions(mc):
    for total in [64, 1000, 10**6, 10**9 + 7]:
        for world in [1, 2, 3, 4, 8]:
            rs = [mc.shard_range(total, r, world) for r in range(world)]
            assert rs[0][0] == 0
            for (b0, c0), (b1, _) in zip(rs, rs[1:]):
                assert b0 + c0 == b1 and b1 % 64 == 0
            assert rs[-1][0] + rs[-1][1] == total


def test_host_surface_matches_oracle_tps(mc, O):
    """The host TPS over arbitrary points (NEXT f2) against the oracle: values, GCV lambda, maximum."""
    rng = np.random.default_rng(0)
    x = rng.uniform(0, 1, (40, 2))
    y = np.exp(-((x - 0.4) ** 2).sum(1) * 3) + 0.01 * rng.normal(size=40)
    for lam in (0.0, 1e-4, -1.0):
        s = mc.Surface(x, y, lam)
        ref, lr = O.tps_smooth(x, y, lam)
        assert s.lam == pytest.approx(lr, rel=1e-12)
        f, _ = s(x)
        assert np.allclose(f, ref, atol=1e-9)
        xs, fs = s.maximum()
        xo, fo, _ = O.refine(x, y, lr)
        assert np.allclose(xs, xo, atol=1e-6) and fs == pytest.approx(fo, abs=1e-9)
    # d = 1 (cubic) as well
    x1 = np.linspace(0, 1, 12)[:, None]
    y1 = np.sin(3 * x1[:, 0])
    s1 = mc.Surface(x1, y1, 0.0)
    assert np.allclose(s1(x1)[0], y1, atol=1e-10)


def test_checkpoint_roundtrip(mc, tmp_path):
    sums = np.arange(20, dtype=np.int64).reshape(10, 2) * (2**40)
    mc.checkpoint_save(str(tmp_path / "ck"), sums, 123456789, 0x2005105494, {"designs": 10})
    s2, done, seed, meta = mc.checkpoint_load(str(tmp_path / "ck"))
    assert np.array_equal(s2, sums) and done == 123456789 and seed == 0x2005105494 and meta["designs"] == 10


def test_grid_smooth_validation_before_device(mc):
    # all argument checks run on the host before any CUDA call (so this runs without a GPU)
    L = mc.lib()
    d = ctypes.c_double
    xr = (d * 4)(0.1, 0.2, 0.3, 0.4)
    bad = (d * 4)(0.1, 0.3, 0.3, 0.4)
    xa = (d * 3)(0.0, 1.0, 2.0)
    fake = ctypes.c_void_p(16)
    assert L.mc_grid_smooth(None, 4, 3, xr, xa, -1.0, -1.0, fake, None, None) == 1
    assert L.mc_grid_smooth(fake, 1, 3, xr, xa, -1.0, -1.0, fake, None, None) == 1
    assert L.mc_grid_smooth(fake, 4, 5000, xr, xa, -1.0, -1.0, fake, None, None) == 1
    assert L.mc_grid_smooth(fake, 4, 3, bad, xa, -1.0, -1.0, fake, None, None) == 1
    assert b"strictly increasing" in L.mc_last_error()
    assert L.mc_grid_smooth(fake, 4, 3, xr, xa, float("inf"), 1.0, fake, None, None) == 1
