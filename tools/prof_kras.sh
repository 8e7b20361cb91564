#!/bin/bash
# paper Kershaw eps=0.05 4th-opt RAS(12,0): launch list after the Schwarz changes, and
# ncu --set full captures of the p=3 local solve (k_schwarz_local_small), the fused
# RAS assembly epilogue (K2 EPI_SUPD4) and the coarse column-dot solve (k_coldot)
mkdir -p gpurun_out
timeout 600 python tools/tts_launches.py --case kras 2>&1 | tail -1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/kras2_launches.csv python tools/tts_launches.py --case kras > gpurun_out/kras2_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/kras2_launches.csv > gpurun_out/kras2_summary.txt 2>&1
for k in 'regex:k_schwarz_local_small' 'regex:k_schwarz_local<' 'regex:k_sem_k2<7, 7>' 'regex:k_coldot'; do
  n=$(echo "$k" | tr -cd 'a-z0-9_')
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "$k" -s 2 -c 1 -o gpurun_out/prof_kras_$n python tools/tts_launches.py --case kras > gpurun_out/ncu_kras_$n.log 2>&1
  echo "ncu $k rc=$?"
done
