"""Count the issue slots per draw of the fused kernel's steady-state loop from its sm_100a SASS.

The steady-state loop of mc_fused_kernel<N, EST> (unmasked per-thread run) is walked from the
target of its backward branch along the COMMON path:
  * `BRA.DIV` (divergence fallback of a warp vote) is not taken;
  * `@!P BRA` right after `VOTE.ANY P` (the warp-uniform rare inverse-CDF tail) is taken, i.e. the
    tail polynomials are skipped;
  * a branch on a predicate last written by `FSETP.GE[U] P, PT, R, {5, 16, 18}` (the inverse-CDF tail
    tests w >= 5, w >= 16, w + 2 >= 18, w + 3 >= 27: rare) goes the common way: `@!P BRA` taken, `@P BRA` not;
  * unconditional forward `BRA` is followed; other conditional forward branches fall through.
Issue slots per draw = path length / draws per iteration.  Used by bench.py for the ALU roofline.

    python tools/sass_count.py [N] [EST]
"""
import collections
import os
import re
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2005_10494_b200", "libmc_design.so")
def draws_per_iter(n: int, est: int, model: int = 0) -> int:
    """L = R * 4 / gcd(WR, 4) samples per Philox-aligned step (mc_device.cuh Geo): records of R = 2 samples
    and U 23-bit uniforms in WR = 2 ceil(23 U / 64) words if that is fewer than U, else U."""
    import math
    p = 5 if model == 1 else n
    R, U = (2, 2 * p + 2 * (n // 2)) if est == 0 else (2, 4 * ((p + n + 1) // 2))
    W = 2 * ((23 * U + 63) // 64)
    WR = W if W < U else U
    return R * (4 // math.gcd(WR, 4))


def sass(n: int, est: int, lib: str = None, model: int = 0):
    out = subprocess.run(["cuobjdump", "-sass", lib or LIB], capture_output=True, text=True).stdout
    # select the function body of mc_fused_kernel<n, est>
    tag = f"_ZN3mci15mc_fused_kernelILi{n}ELi{est}ELi{model}EEEv"
    lines, on = [], False
    for line in out.splitlines():
        if "Function :" in line:
            on = tag in line
        elif on:
            lines.append(line)
    out = "\n".join(lines)
    ins = []
    for line in out.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    return ins


def _target(text):
    m = re.search(r"\bBRA(?:\.\w+)?\s+(?:U?P\w+,\s*)?(?:UR\w+,\s*)?0x([0-9a-f]+)", text)
    return int(m.group(1), 16) if m else None


def walk(ins, start, end):
    """Common path from address `start` until the back edge at `end`."""
    idx = {a: i for i, (a, _) in enumerate(ins)}
    i = idx[start]
    path = []
    prev = ""
    rare = {}          # predicate -> True if last written by a rare-tail FSETP
    for _ in range(20000):
        a, t = ins[i]
        path.append((a, t))
        if a == end:
            break
        m = re.match(r"FSETP\.(\w+)\.AND (P\d), PT, [^,]+, ([0-9.e+-]+), PT", t)
        if m:
            rare[m.group(2)] = m.group(1) in ("GE", "GEU") and float(m.group(3)) in (5.0, 16.0, 18.0, 27.0)
        else:
            m = re.match(r"\w+(?:\.\w+)* (P\d),", t)
            if m and not t.startswith("@"):
                rare[m.group(1)] = False
        tgt = _target(t)
        pm = re.match(r"@(!?)(P\d) BRA", t)
        if tgt is not None and "BRA" in t:
            if "BRA.DIV" in t:
                i += 1
            elif t.startswith("@!P") and prev.startswith("VOTE.ANY P"):
                i = idx[tgt]
            elif pm and rare.get(pm.group(2)):
                i = idx[tgt] if pm.group(1) == "!" else i + 1
            elif t.startswith("@P") and ("FSETP.GEU" in prev and (", 5," in prev or ", 16," in prev)):
                i += 1          # w >= 5 / w >= 16: the inverse-CDF tails, not taken on the common path
            elif not t.startswith("@") and tgt > a:
                i = idx[tgt]
            else:
                i += 1
        else:
            i += 1
        if i >= len(ins):
            break
        prev = t
    return path


def steady_loop(ins):
    """The innermost sample loop: the shortest back-edge cycle that evaluates draws (has MUFU) and
    contains no block barrier (which marks the outer tile loop); the masked variant is longer."""
    best = None
    for a, t in ins:
        tgt = _target(t)
        if tgt is not None and tgt < a and "BRA" in t:
            p = walk(ins, tgt, a)
            if p[-1][0] != a or any(x.startswith("BAR") for _, x in p):
                continue
            if not any(x.startswith("MUFU") for _, x in p):
                continue
            if best is None or len(p) < len(best):
                best = p
    return best


def issue_per_draw(n: int = 3, est: int = 0, lib: str = None) -> float:
    return len(steady_loop(sass(n, est, lib))) / draws_per_iter(n, est)


FP32_OPS = ("FFMA", "FMUL", "FADD")       # the FP32 (FMA) pipe's arithmetic
FP32X2_OPS = ("FFMA2", "FMUL2", "FADD2")  # packed pairs: one issue slot, two FP32 lane-ops
SFU_OPS = ("MUFU",)


# sm_100a per-SMSP pipe model, measured on this pool's B200 (tools/pipemix.cu + ncu pipe counters,
# profiles/r02/pipe_model.md): cycles one warp-instruction occupies each unit.
#   FFMA2/FMUL2/FADD2   fmaheavy 2 AND fmalite 2      FFMA/FMUL/FADD   fmaheavy 2 OR fmalite 2
#   IMAD (32-bit)       fmaheavy 2                     IMAD.WIDE        fmaheavy 4
#   LOP3/FMNMX/FSEL/FSETP/IADD3/MOV/SHF/...  alu 2     MUFU / F2F       xu 8
# and one issue slot per instruction.
ALU_OPS = ("LOP3", "FMNMX", "FMNMX3", "FSEL", "FSETP", "ISETP", "IADD3", "MOV", "SHF", "SEL", "PRMT", "LEA",
           "VIADD", "IADD", "FLO", "POPC", "VIMNMX")


def pipe_mix(n: int = 3, est: int = 0, lib: str = None, model: int = 0) -> dict:
    """Per-draw counts of the executed common path by pipe class: issue slots, FP32 lane-ops (FFMA/FMUL/FADD;
    packed x2 count twice), SFU (MUFU), IMAD.WIDE (the Philox multiplies), and the per-WARP-draw cycles of
    each unit under the measured pipe model (scalar FP32 placed on fmalite, i.e. the fmaheavy lower bound)."""
    path = steady_loop(sass(n, est, lib, model))
    L = draws_per_iter(n, est, model)
    ops = [(t.split()[1] if t.startswith("@") else t.split()[0]) for _, t in path]
    base = [o.split(".")[0] for o in ops]
    p2 = sum(b in FP32X2_OPS for b in base)
    sc = sum(b in FP32_OPS for b in base)
    wide = sum(o.startswith("IMAD.WIDE") for o in ops)
    imad = sum(b == "IMAD" for b in base) - wide
    alu = sum(b in ALU_OPS for b in base)
    xu = sum(b in SFU_OPS or b == "F2F" for b in base)
    return {"issue": len(path) / L,
            "fp32": (sc + 2 * p2) / L,
            "sfu": sum(b in SFU_OPS for b in base) / L,
            "imad_wide": wide / L,
            "cycles": {"issue": len(path) / L, "fmaheavy": (2 * p2 + 4 * wide + 2 * imad) / L,
                       "fmalite": (2 * p2 + 2 * sc) / L, "alu": 2 * alu / L, "xu": 8 * xu / L}}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    est = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    path = steady_loop(sass(n, est))
    L = draws_per_iter(n, est)
    op = collections.Counter((t.split()[1] if t.startswith("@") else t.split()[0]).split(".")[0] for _, t in path)
    print(f"mc_fused_kernel<{n},{est}>: common path {len(path)} instr, {L} draws/iteration -> "
          f"{len(path) / L:.1f} issue slots/draw")
    for k, v in op.most_common():
        print(f"  {k:12s} {v:4d}  ({v / L:.1f}/draw)")


if __name__ == "__main__":
    main()
