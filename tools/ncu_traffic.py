"""Sum DRAM traffic of the K1/K2 launches of ONE sweep from an ncu report
(tools/one_sweep.py under ncu --profile-from-start off) and write
profiles/r02/sem_sweep_traffic.json for bench.py's roofline.traffic.

    python tools/ncu_traffic.py REPORT.ncu-rep [--E 64] [--order 8]
"""
import argparse
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def num(v):
    return float(v.replace(",", "")) if v not in ("", "n/a") else 0.0


ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--E", type=int, default=64)
ap.add_argument("--order", type=int, default=8)
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "sem_sweep_traffic.json"))
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
tscale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
per = []
for r in rows[2:]:
    d = dict(zip(h, r))
    u = dict(zip(h, units))
    name = d.get("Kernel Name", "")
    rd = num(d["dram__bytes_read.sum"]) * scale.get(u["dram__bytes_read.sum"], 1)
    wr = num(d["dram__bytes_write.sum"]) * scale.get(u["dram__bytes_write.sum"], 1)
    t = num(d["gpu__time_duration.sum"]) * tscale.get(u["gpu__time_duration.sum"], 1e-9)
    per.append({"kernel": name[:90], "dram_bytes": rd + wr, "time_s": t})
sem_k = [p for p in per if "k_sem_k1" in p["kernel"] or "k_sem_k2" in p["kernel"]]
E, order = a.E, a.order
n = (7 * E - 1) ** 3
alg = order * 48 * 512 * E ** 3 + (40 + 64 * (order - 2) + 48) * n
dram = sum(p["dram_bytes"] for p in sem_k)
res = {"source": os.path.basename(a.report) + " (tools/one_sweep.py, one order-%d sweep)" % order,
       "elements": E ** 3, "order": order, "launches": len(sem_k), "dram_bytes_per_sweep": dram,
       "algorithmic_bytes_per_sweep": alg, "ratio": dram / alg,
       "kernel_time_s": sum(p["time_s"] for p in sem_k), "all_launches": per}
os.makedirs(os.path.dirname(a.out), exist_ok=True)
with open(a.out, "w") as fh:
    json.dump(res, fh, indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "all_launches"}, indent=1))
