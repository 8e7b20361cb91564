#!/bin/bash
# same-box A/B of the fused CGS pass on the SEM time-to-solution; RAS launch list
mkdir -p gpurun_out
for rep in 1 2; do
  for val in 0 1; do
    CMG_CGS_FUSE=$val timeout 300 python tools/tts_launches.py --case sem 2>&1 | tail -1 | sed "s/^/FUSE=$val /"
  done
done
timeout 300 python tools/tts_launches.py --case ras > gpurun_out/tts_plain_ras.log 2>&1 && \
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  --csv --log-file gpurun_out/tts_launches_ras.csv python tools/tts_launches.py --case ras > /dev/null 2>&1
cat gpurun_out/tts_plain_ras.log
python tools/launch_summary.py gpurun_out/tts_launches_ras.csv | head -16
