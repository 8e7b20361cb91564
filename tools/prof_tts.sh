#!/bin/bash
# launch lists of one SEM p-MG-PGMRES solve (E=64) and one FD config-1 solve
mkdir -p gpurun_out
timeout 300 python tools/tts_launches.py --case sem > gpurun_out/tts_plain_sem.log 2>&1 || exit 1
timeout 300 python tools/tts_launches.py --case fd > gpurun_out/tts_plain_fd.log 2>&1 || exit 1
for c in sem fd; do
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --kernel-name-base demangled --csv --log-file gpurun_out/tts_launches_$c.csv \
      python tools/tts_launches.py --case $c > gpurun_out/tts_ncu_$c.log 2>&1
done
cat gpurun_out/tts_plain_*.log
echo done
