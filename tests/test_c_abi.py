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


def test_ctypes_mc_problem_layout_matches_header(tmp_path):
    """mc.py declares mc_problem by hand for ctypes: its size and every field offset must
    equal what a C compiler lays out from include/mc_design.h."""
    import ctypes
    from paper_2005_10494_b200 import mc
    fields = [f[0] for f in mc.mc_problem._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "mc_design.h"\nint main(void) {\n'
                   '  printf("size %zu\\n", sizeof(mc_problem));\n'
                   + "".join(f'  printf("{f} %zu\\n", offsetof(mc_problem, {f}));\n' for f in fields)
                   + "  return 0;\n}\n")
    cc = shutil.which("cc") or shutil.which("gcc")
    exe = str(tmp_path / "layout")
    subprocess.run([cc, "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", exe], check=True)
    out = dict(line.split() for line in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.splitlines())
    assert int(out["size"]) == ctypes.sizeof(mc.mc_problem)
    for f in fields:
        assert int(out[f]) == getattr(mc.mc_problem, f).offset, f
