#!/bin/bash
# same-box A/B of the fused CGS pass on the SEM time-to-solution (+ kernel durations)
mkdir -p gpurun_out
for rep in 1 2 3; do
  for val in 0 1; do
    CMG_CGS_FUSE=$val timeout 300 python tools/tts_launches.py --case sem 2>&1 | tail -1 | sed "s/^/FUSE=$val /"
  done
done
for val in 0 1; do
  CMG_CGS_FUSE=$val timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
    -k 'regex:k_layer|k_cgs' --csv --log-file gpurun_out/ab_cgs_$val.csv python tools/tts_launches.py --case sem > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/ab_cgs_$val.csv | head -6 | sed "s/^/FUSE=$val /"
done
