"""The boundary as a C program sees it: tests/c_abi/c1_abi.c is compiled with the system C
compiler against include/mc_design.h alone and linked to libmc_design.so.  The build and link run on CPU;
running it (C1 through init -> evaluate -> finalize -> argmax, checked against the oracle's stored output
tests/golden/c1_oracle_1e4.txt) needs the GPU."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c_abi", "c1_abi.c")
CUDA = "/usr/local/cuda"


def _compile(tmp_path):
    from paper_2005_10494_b200 import build
    build.build()
    cc = shutil.which("cc") or shutil.which("gcc")
    exe = str(tmp_path / "c1_abi")
    libdir = os.path.dirname(build.LIB)
    cmd = [cc, "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include", SRC,
           "-L", libdir, "-lmc_design", "-L", f"{CUDA}/lib64", "-lcudart", "-lm",
           f"-Wl,-rpath,{libdir}", f"-Wl,-rpath,{CUDA}/lib64", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_program_compiles_and_links(tmp_path):
    exe = _compile(tmp_path)
    assert os.path.exists(exe)
    # every undefined mc_* symbol of the program resolves in the library
    nm = subprocess.run(["nm", "-u", exe], capture_output=True, text=True).stdout
    used = {ln.split()[-1] for ln in nm.splitlines() if ln.split() and ln.split()[-1].startswith("mc_")}
    assert {"mc_design_init", "mc_evaluate_grid", "mc_finalize", "mc_argmax"} <= used


@pytest.mark.gpu
def test_c_program_c1_matches_oracle(tmp_path):
    exe = _compile(tmp_path)
    r = subprocess.run([exe, os.path.join(ROOT, "tests", "golden", "c1_oracle_1e4.txt")], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
