#!/bin/bash
# Same-box A/B of two library builds (the bench sweep only):
#   bash tools/ab_lib.sh path/to/A.so path/to/B.so [reps]
A=$1; B=$2; REPS=${3:-3}
mkdir -p gpurun_out
for rep in $(seq $REPS); do
  for L in $A $B; do
    CMG_LIB=$L timeout 300 python bench.py --no-cpu --no-solve --no-configs --steps 20 > gpurun_out/ab_lib.log 2>&1
    python - "$L" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab_lib.log").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"], 3), round(d["roofline"]["frac"], 4), d["step_ms_min_max"], d["clocks"]["sm_mhz"])
PY
  done
done
