"""Instruction mix of the warp-specialised K1 loops (mc_ws_kernel, the round-2 experiment in
profiles/r02/k1_ws_experiment.patch — measured slower, not shipped) from a library built with that patch:
the producer's Philox loop and the consumer's evaluation loop (tuning aid).

    python tools/ws_loops.py [LIB] [N] [EST]
"""
import collections
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import sass_count as s  # noqa: E402


def sass_fn(lib, tag):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    lines, on = [], False
    for line in out.splitlines():
        if "Function :" in line:
            on = tag in line
        elif on:
            lines.append(line)
    ins = []
    for line in lines:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    return ins


def loops(lib, n=3, est=0):
    ins = sass_fn(lib, f"_ZN3mci12mc_ws_kernelILi{n}ELi{est}EEE")
    res = []
    for a, t in ins:
        tgt = s._target(t)
        if tgt is not None and tgt < a and "BRA" in t:
            p = s.walk(ins, tgt, a)
            if p[-1][0] != a:
                continue
            ops = collections.Counter((t.split()[1] if t.startswith("@") else t.split()[0]) for _, t in p)
            res.append((tgt, a, len(p), ops))
    return res


if __name__ == "__main__":
    lib = sys.argv[1] if len(sys.argv) > 1 else s.LIB
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    est = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    for tgt, a, ln, ops in loops(lib, n, est):
        g = lambda pre: sum(v for k, v in ops.items() if k.startswith(pre))
        if g("SYNCS") and (g("MUFU") or g("IMAD.WIDE")) and not g("LDL") + g("STL") > 20:
            print(f"{tgt:#x}-{a:#x}: {ln} instr, MUFU {g('MUFU')}, IMAD.WIDE {g('IMAD.WIDE')}, "
                  f"LDS/STS {g('LDS') + g('STS')}, SYNCS {g('SYNCS')}, LDL/STL {g('LDL') + g('STL')}")
