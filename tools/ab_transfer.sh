#!/bin/bash
# transfers A/B (same box): per-kernel launch times of one E=64^3 solve and the bench TTS
mkdir -p gpurun_out
for v in 2 1 0; do
  CMG_TRANSFER_KERNEL=$v timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name-base demangled -k 'regex:k_prolong|k_restrict' --csv \
    --log-file gpurun_out/transfer_tma$v.csv python tools/one_sweep.py --solve > gpurun_out/transfer_tma$v.log 2>&1
  python3 - "$v" <<'PY'
import csv, sys, collections
v = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/transfer_tma{v}.csv")))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]; d = rows[i + 1:]
K, M, V = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in d:
    agg[r[K][:60]][r[M]].append(float(r[V].replace(",", "")))
for k, m in agg.items():
    t = sum(m["gpu__time_duration.sum"]) / len(m["gpu__time_duration.sum"])
    b = (sum(m["dram__bytes_read.sum"]) + sum(m["dram__bytes_write.sum"])) / len(m["gpu__time_duration.sum"])
    print(f"K={v} {k}: {t/1e3:.1f} us, {b/1e9:.3f} GB, {b/(t*1e-9)/1e9:.0f} GB/s")
PY
done
for rep in 1 2; do for v in 2 0; do
  CMG_TRANSFER_KERNEL=$v timeout 300 python bench.py --no-cpu --no-configs --steps 5 > gpurun_out/ab_tr.log 2>&1
  python3 -c "
import json; d=json.loads(open('gpurun_out/ab_tr.log').read().strip().splitlines()[-1]); print('K=$v', 'TTS', d['time_to_solution']['time_to_solution_s'], d['time_to_solution']['iterations'])"
done; done
