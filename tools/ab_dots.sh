#!/bin/bash
# multi-dot / fused-CGS unroll A/B (E=64^3 solve): per-kernel time + TTS
mkdir -p gpurun_out
for cfg in "4 1" "4 2" "4 3"; do set -- $cfg
  CMG_DOTS_UNROLL=$1 CMG_CGS_UNROLL=$2 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base demangled --profile-from-start off -k 'regex:k_layer_dots|k_layer_cgs_dots' \
    --csv --log-file gpurun_out/dots_$1_$2.csv python tools/one_sweep.py --solve > /dev/null 2>&1
  python3 - "$1_$2" <<'PY'
import csv, collections, sys
rows = list(csv.reader(open(f"gpurun_out/dots_{sys.argv[1]}.csv")))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]; d = rows[i + 1:]
ID, K, M, V = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = collections.defaultdict(dict)
for r in d:
    per[(r[ID], r[K][:46])][r[M]] = float(r[V].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (idx, k), m in per.items():
    a = agg[k]; a[0] += 1; a[1] += m["gpu__time_duration.sum"]; a[2] += m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"D/C={sys.argv[1]} {n:3d} {t/1e3:9.1f} us {b/(t*1e-9)/1e12:5.2f} TB/s {k}")
PY
done
for rep in 1 2; do for cfg in "4 2" "1 1"; do set -- $cfg
  CMG_DOTS_UNROLL=$1 CMG_CGS_UNROLL=$2 timeout 600 python tools/tts_config.py --E 64 --smoother 0 --kpre 8 --kpost 0 --reps 3 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('D/C=$1_$2 TTS', d['tts_ms'], d['iterations'])"
done; done
