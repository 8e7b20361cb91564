#!/bin/bash
# same-box A/B of library builds on the E=64^3 time to solution (+ sweep):
#   bash tools/ab_tts_lib.sh a.so b.so [reps]
A=$1; B=$2; REPS=${3:-2}
mkdir -p gpurun_out
for rep in $(seq $REPS); do for L in $A $B; do
  CMG_LIB=$L timeout 600 python bench.py --no-cpu --no-configs --steps 10 > gpurun_out/ab_tts.log 2>&1
  python3 -c "
import json; d=json.loads(open('gpurun_out/ab_tts.log').read().strip().splitlines()[-1])
print('$L', round(d['value'],2), 'TTS', d['time_to_solution']['time_to_solution_s'], d['clocks']['sm_mhz'])"
done; done
