"""Text summary of one-kernel ncu --set full reports: duration, DRAM bytes and
rate, L1/shared pipe, occupancy, warp-stall breakdown (whole kernel and per
barrier-delimited phase of the SASS) and the top stalled source lines.

    python tools/ncu_summary.py REPORT.ncu-rep [...] > profiles/r02/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs)"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem)"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
]
STALLS = ["stall_long_sb", "stall_wait", "stall_short_sb", "stall_barrier", "stall_mio", "stall_lg", "stall_math",
          "stall_not_selected", "stall_selected", "stall_dispatch", "stall_branch_resolving", "stall_membar"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


for rep in sys.argv[1:]:
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u = raw[0], raw[1]
    for row in raw[2:]:
        d = dict(zip(h, row))
        un = dict(zip(h, u))
        print(f"# {d.get('Kernel Name', '?')[:100]}  ({rep.split('/')[-1]})")
        for k, name in KEYS:
            if k in d:
                print(f"  {name:26s} {d[k]} {un.get(k, '')}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    if len(src) < 3:
        continue
    sh = src[1]
    iS, isrc = sh.index("Warp Stall Sampling (All Samples)"), sh.index("Source")

    def num(v):
        try:
            float(v or 0)
            return True
        except ValueError:
            return False
    # multi-kernel reports repeat the header per kernel: keep the first kernel's rows
    rows = []
    for x in src[2:]:
        if len(x) <= iS or not num(x[iS]):
            break
        rows.append(x)
    ic = {c: sh.index(c) for c in STALLS if c in sh}
    tot = sum(float(x[iS] or 0) for x in rows) or 1.0
    allst = {c: sum(float(x[i] or 0) for x in rows if len(x) > i) / tot * 100 for c, i in ic.items()}
    print("  stalls (% of samples): " + ", ".join(f"{c[6:]} {v:.0f}" for c, v in sorted(allst.items(), key=lambda kv: -kv[1]) if v >= 1))
    reg, acc = 0, {}
    for x in rows:
        acc.setdefault(reg, [0.0, 0])
        acc[reg][0] += float(x[iS] or 0)
        acc[reg][1] += 1
        if "BAR.SYNC" in x[isrc]:
            reg += 1
    print("  samples per barrier-delimited phase: " + ", ".join(f"{k}:{v[0] / tot * 100:.0f}%" for k, v in acc.items()))
    top = sorted(rows, key=lambda x: -float(x[iS] or 0))[:6]
    for x in top:
        st = max(ic, key=lambda c: float(x[ic[c]] or 0) if len(x) > ic[c] else 0.0)
        print(f"    {float(x[iS]) / tot * 100:5.1f}%  {x[isrc].strip()[:60]:60s} ({st[6:]})")
