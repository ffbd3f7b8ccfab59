"""Count the issue slots per draw of the fused kernel's steady-state loop from its sm_100a SASS.

The unmasked per-thread loop of mc_fused_kernel<N, EST> is the block ending in the backward branch
with the largest body.  Inside it, every inverse-normal-CDF call has a three-way branch (central,
tail, deep tail); the common path takes the central polynomial, so the tail blocks are subtracted.
Prints the opcode histogram and issue slots per draw (used as bench.py ISSUE_PER_DRAW).

    python tools/sass_count.py [N] [EST]
"""
import collections
import re
import subprocess
import sys

LIB = "paper_2005_10494_b200/libmc_design.so"


def sass(n: int, est: int):
    sym = f"_ZN3mci15mc_fused_kernelILi{n}ELi{est}EEEvPKfS2_PKilmmmllmPy"
    out = subprocess.run(["cuobjdump", "-sass", "-fun", sym, LIB], capture_output=True, text=True).stdout
    ins = []
    for line in out.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    return ins


def loop_body(ins):
    best = None
    for addr, text in ins:
        m = re.search(r"\bBRA\s+(?:\w+,\s*)?0x([0-9a-f]+)", text)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < addr and (best is None or addr - tgt > best[1] - best[0]):
                best = (tgt, addr)
    lo, hi = best
    return [(a, t) for a, t in ins if lo <= a <= hi]


def common_path(body):
    """Drop the tail branches of the quantile: from each `FMNMX Rx, Ry, 88` (tail entry) up to the
    join target of the preceding central block's BRA."""
    keep = []
    skip_until = None
    for i, (a, t) in enumerate(body):
        if skip_until is not None:
            if a < skip_until:
                continue
            skip_until = None
        if t.startswith("FMNMX") and ", 88" in t:
            # the central block ends with `BRA join` just before this instruction
            prev = body[i - 1][1]
            m = re.search(r"BRA\s+0x([0-9a-f]+)", prev)
            skip_until = int(m.group(1), 16)
            keep.pop()   # the central block's BRA is not executed as a taken jump on the fall-through path
            keep.append((body[i - 1][0], "BRA(central->join)"))
            continue
        keep.append((a, t))
    return keep


DRAWS_PER_ITER = {0: {1: 2, 2: 4, 3: 2}, 1: {1: 2, 2: 1, 3: 2}}


def issue_per_draw(n: int = 3, est: int = 0, lib: str = None) -> float:
    """Common-path issue slots per draw of mc_fused_kernel<n, est> in the built library."""
    global LIB
    if lib:
        LIB = lib
    path = common_path(loop_body(sass(n, est)))
    return len(path) / DRAWS_PER_ITER[est][n]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    est = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    ins = sass(n, est)
    body = loop_body(ins)
    path = common_path(body)
    L = DRAWS_PER_ITER.get(est, {}).get(n, 2)
    op = collections.Counter(t.split()[0].lstrip("@!P0123456789T ").split(".")[0] if not t.startswith("@")
                             else t.split()[1].split(".")[0] for _, t in path)
    print(f"mc_fused_kernel<{n},{est}>: loop body {len(body)} instr, common path {len(path)} instr, "
          f"{L} draws/iteration -> {len(path) / L:.1f} issue slots/draw")
    for k, v in op.most_common():
        print(f"  {k:12s} {v:4d}  ({v / L:.1f}/draw)")


if __name__ == "__main__":
    main()
