#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sem_gpu.py -m gpu -q -x -k "not full_size" > gpurun_out/tr_tests.log 2>&1; echo "sem tests rc=$?"; tail -1 gpurun_out/tr_tests.log
for i in 1 2; do timeout 300 python tools/tts_launches.py --case sem 2>&1 | tail -1; done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k 'regex:k_prolong|k_restrict' --csv --log-file gpurun_out/tr_launch.csv python tools/tts_launches.py --case sem > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/tr_launch.csv | head -8
