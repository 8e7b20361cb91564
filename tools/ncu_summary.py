"""One-line summaries of ncu --set full reports (duration, DRAM bytes, occupancy, stalls)."""
import csv
import subprocess
import sys

for f in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    for vals in r[2:]:
        d = {h[i]: vals[i] for i in range(len(h))}
        u = {h[i]: units[i] for i in range(len(h))}
        def g(k):
            return f"{d.get(k)} {u.get(k, '')}".strip()
        print(f"{f}: {d.get('Kernel Name', '')[:70]}")
        print(f"  duration {g('gpu__time_duration.sum')}  dram read {g('dram__bytes_read.sum')}  write "
              f"{g('dram__bytes_write.sum')}  dram% {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')}")
        print(f"  regs {g('launch__registers_per_thread')}  occupancy {g('sm__warps_active.avg.pct_of_peak_sustained_active')}"
              f"  block {g('launch__block_size')}  smem/block {g('launch__shared_mem_per_block_dynamic')}")
        keys = [k for k in h if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
        st = sorted([(float(d[k].replace(",", "")), k) for k in keys if d[k] not in ("", "n/a")], reverse=True)
        tot = sum(v for v, _ in st) or 1.0
        print("  stalls: " + ", ".join(f"{k.split('stalled_')[1]} {100 * v / tot:.0f}%" for v, k in st[:7]))
