#!/bin/bash
mkdir -p gpurun_out
for v in 1 0; do
  CMG_SCHWARZ_IL=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
    --kernel-name-base demangled -k 'regex:k_schwarz_local' -c 6 --csv --log-file gpurun_out/schwarz_il$v.csv \
    python tools/tts_config.py --E 32 --smoother 2 --kpre 1 --kpost 1 --reps 1 > /dev/null 2>&1
  grep -h "k_schwarz_local" gpurun_out/schwarz_il$v.csv | awk -F'","' '{print "IL='$v'", $5, $(NF)}' | cut -c1-120
done
for rep in 1 2; do for v in 1 0; do
  CMG_SCHWARZ_IL=$v python tools/tts_config.py --E 32 --smoother 2 --kpre 1 --kpost 1
  CMG_SCHWARZ_IL=$v python tools/tts_config.py --E 32 --smoother 1 --kpre 2 --kpost 0
done; done
