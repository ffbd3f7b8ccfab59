"""Summarise ncu output for profiles/ (run here, on the CPU side, after gpurun brought the files back).

    python tools/ncu_summary.py launches LAUNCHES.csv "command" > profiles/rNN/ncu_launches_summary.txt
    python tools/ncu_summary.py report REPORT.ncu-rep "title" > profiles/rNN/ncu_fused_cond_summary.txt

`launches`: per-kernel totals and shares of a `--metrics gpu__time_duration.sum --csv` launch list (the
kernels that run every step, and all launches).  `report`: the key metrics of a `--set full` capture
(issue, pipes, stalls per issue, occupancy, DRAM bytes, clock) via `ncu -i ... --page raw --csv`.
"""
import collections
import csv
import io
import re
import subprocess
import sys

STEP_KERNELS = ("mc_fused_kernel", "mc_crn_kernel", "k_e_c", "k_gcv", "k_et_y", "k_segmented_argmax", "k_gather",
                "k_finalize", "k_zc")


def _short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name).strip()
    return name[:80]


def launches(path: str, title: str):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v *= {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1.0}.get(unit, 1.0)
        k = _short(r["Kernel Name"])
        tot[k][0] += 1
        tot[k][1] += v
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none) of: {title}")
    print("# cold-cache, serialised per-launch times: compare SHARES.\n")
    for label, keep in (("per-step kernels only", lambda k: any(s in k for s in STEP_KERNELS)),
                        ("all launches incl. one-time prep", lambda k: True)):
        sel = {k: v for k, v in tot.items() if keep(k)}
        s = sum(v[1] for v in sel.values()) or 1.0
        print(f"## {label}")
        print(f"{'kernel':82s} {'launches':>8s} {'total_ns':>14s} {'share':>7s}")
        for k, (n, t) in sorted(sel.items(), key=lambda kv: -kv[1][1])[:25]:
            print(f"{k:82s} {n:8d} {t:14.0f} {100 * t / s:6.2f}%")
        print()


KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "sm__warps_active.avg.per_cycle_active",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]


def report(path: str, title: str):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# {title}")
    for v in rows[2:]:
        print(f"## {_short(v[h.index('Kernel Name')])}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"{k:78s} {v[i]:>22s} {units[i]}")
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                if v[i] not in ("", "0") and float(v[i]) >= 0.001:
                    print(f"{k:78s} {v[i]:>22s}")
        print()


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[2])
