#!/bin/bash
# fused K1+K2 step: SEM parity tests with it (under a hard timeout), then same-box A/B
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_sem_gpu.py -m gpu -q -x -k "not full_size" > gpurun_out/fused_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/fused_tests.log
for rep in 1 2; do
  for val in 0 1; do
    CMG_SEM_FUSED=$val timeout 300 python bench.py --no-cpu > gpurun_out/ab_fused_$val.log 2>&1
    echo "rc=$?"
    tail -1 gpurun_out/ab_fused_$val.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('FUSED=$val', round(d['value'],2), round(d['roofline']['frac'],4), d['step_ms_min_max'], 'tts', d['time_to_solution']['time_to_solution_s'], d['time_to_solution']['iterations'])"
  done
done
