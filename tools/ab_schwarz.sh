#!/bin/bash
# DMMA Schwarz local solve: parity tests, then same-box A/B of the RAS solve and the kernel
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_sem_gpu.py -m gpu -q -x -k "schwarz" > gpurun_out/schwarz_tests.log 2>&1; echo "schwarz tests (mma) rc=$?"; tail -1 gpurun_out/schwarz_tests.log
for rep in 1 2; do for val in 0 1; do
  CMG_SCHWARZ_MMA=$val timeout 300 python tools/tts_launches.py --case ras 2>&1 | tail -1 | sed "s/^/MMA=$val /"
done; done
for val in 0 1; do
  CMG_SCHWARZ_MMA=$val timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
    -k 'regex:k_schwarz_local' -s 4 -c 4 --csv --log-file gpurun_out/ab_sch_$val.csv python tools/tts_launches.py --case ras > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/ab_sch_$val.csv | head -4 | sed "s/^/MMA=$val /"
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:k_schwarz_local_mma<.int.7>' -s 2 -c 1 -o gpurun_out/prof_schwarz_mma python tools/tts_launches.py --case ras > /dev/null 2>&1
echo "ncu rc=$?"
