#!/bin/bash
# timing probe of the fused-step variants (CMG_FUSED_MODE) vs the two-kernel step
mkdir -p gpurun_out
run() {
  env "$@" timeout 240 python bench.py --no-cpu --no-solve > gpurun_out/ab_fm.log 2>&1
  rc=$?
  echo -n "$* rc=$rc "
  tail -1 gpurun_out/ab_fm.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), d['step_ms_min_max'])" 2>/dev/null || echo
}
run CMG_SEM_FUSED=0
run CMG_SEM_FUSED=1 CMG_FUSED_MODE=3
run CMG_SEM_FUSED=1 CMG_FUSED_MODE=4
run CMG_SEM_FUSED=1 CMG_FUSED_MODE=5
run CMG_SEM_FUSED=1 CMG_FUSED_MODE=0
