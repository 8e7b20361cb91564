#!/bin/bash
# A/B a K1 variant knob on the GPU box:
#   bash tools/ab_env.sh VAR "v1 v2 ..." [TESTVAL]
# runs the SEM GPU tests with VAR=TESTVAL (if given), then the bench (no CPU
# baseline, no solve) twice per value, printing value / roofline frac / step ms.
V=${1:-CMG_K1_GREG}
VALS=${2:-"0 1"}
mkdir -p gpurun_out
if [ -n "$3" ]; then
  env $V=$3 timeout 400 python -m pytest tests/test_sem_gpu.py -m gpu -q -x > gpurun_out/ab_tests.log 2>&1
  echo "tests($V=$3) rc=$?"; tail -1 gpurun_out/ab_tests.log
fi
for rep in 1 2; do
  for val in $VALS; do
    env $V=$val timeout 300 python bench.py --no-cpu --no-solve > gpurun_out/ab_$val.log 2>&1
    python - "$val" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"], 3), round(d["roofline"]["frac"], 4), d["step_ms_min_max"])
PY
  done
done
