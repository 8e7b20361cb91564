#!/bin/bash
# Schwarz (RAS) smoother: parity tests, one RAS solve, kernel duration of the local FDM solve
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_sem_gpu.py -m gpu -q -x -k "schwarz" > gpurun_out/schwarz_tests.log 2>&1; echo "schwarz tests rc=$?"; tail -1 gpurun_out/schwarz_tests.log
timeout 300 python tools/tts_launches.py --case ras 2>&1 | tail -1
timeout 300 python tools/tts_launches.py --case ras 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:k_schwarz_local<.int.7>' -s 2 -c 1 -o gpurun_out/prof_schwarz python tools/tts_launches.py --case ras > gpurun_out/ncu_schwarz.log 2>&1
echo "ncu rc=$?"
