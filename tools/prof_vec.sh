#!/bin/bash
# DRAM bytes and duration of the Krylov / vector kernels of one E=64^3 solve
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --kernel-name-base demangled --profile-from-start off \
  -k 'regex:k_layer_dots|k_layer_cgs_dots|k_cgs_update|k_form_iterate|k_normalize_if_pos|k_cheb4_init_zero|k_layer_reduce' \
  --csv --log-file gpurun_out/vec_kernels.csv python tools/one_sweep.py --solve > /dev/null 2>&1
python3 - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/vec_kernels.csv")))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]; d = rows[i + 1:]
ID, K, M, V = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = collections.defaultdict(dict)
for r in d:
    per[(r[ID], r[K][:50])][r[M]] = float(r[V].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (idx, k), m in per.items():
    a = agg[k]; a[0] += 1; a[1] += m["gpu__time_duration.sum"]; a[2] += m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:4d} {t/1e3:9.1f} us {b/1e9:7.2f} GB {b/(t*1e-9)/1e12:6.2f} TB/s  {k}")
PY
