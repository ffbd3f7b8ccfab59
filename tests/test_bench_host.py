"""Host-side pieces of bench.py (no GPU): the reference arm's JSON line (the driver runs
`bench.py --impl reference` and computes its ratio from it), the roofline arithmetic, and that the
committed pipe-mix fallback (used when cuobjdump is absent on the box) is the mix of the library built here."""
import json
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def test_reference_arm_json_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                          "--draws", "20000"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "MC draws/sec (design x sample)" and d["unit"] == "draws/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["steps"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "draws/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_kernel_roofline_arithmetic():
    import bench
    mix = bench.PIPE_MIX_FALLBACK["cond"]
    f, sms = 1.965e9, 148
    bound = 4 * sms * f * 32 / mix["cycles"]["fmaheavy"]
    r = bench.kernel_roofline(mix, 0.5 * bound, sms, f)
    assert r["pipe"] == "fmaheavy" and r["bound"] == "alu"
    assert abs(r["bound_draws_per_s"] - bound) < 1e-3 * bound
    assert abs(r["frac"] - 0.5) < 1e-4 and abs(r["achieved"] / r["peak"] - 0.5) < 1e-3
    assert abs(r["pipes"]["fmaheavy"]["frac"] - 0.5) < 1e-4
    # every other unit's fraction scales with its cycles
    for u, c in mix["cycles"].items():
        assert abs(r["pipes"][u]["frac"] - 0.5 * c / mix["cycles"]["fmaheavy"]) < 1e-4, u


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="needs cuobjdump")
@pytest.mark.parametrize("est", ["cond", "ind"])
def test_pipe_mix_fallback_matches_built_library(est):
    import bench
    import sass_count
    lib = os.path.join(ROOT, "paper_2005_10494_b200", "libmc_design.so")
    if not os.path.exists(lib):
        pytest.skip("library not built")
    got = sass_count.pipe_mix(3, 0 if est == "cond" else 1, lib)
    ref = bench.PIPE_MIX_FALLBACK[est]
    for k in ("issue", "fp32", "sfu", "imad_wide"):
        assert got[k] == pytest.approx(ref[k]), k
    for u, c in ref["cycles"].items():
        assert got["cycles"][u] == pytest.approx(c), u
