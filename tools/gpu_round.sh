#!/bin/bash
# FD + SEM parity tests, bench line, FD/SEM time-to-solution, BASELINE config table
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fd_gpu.py tests/test_sem_gpu.py -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python tools/tts_launches.py --case fd
timeout 300 python tools/tts_launches.py --case fd
timeout 300 python bench.py --no-cpu > gpurun_out/bench_quick.log 2>&1
echo "bench rc=$?"; tail -1 gpurun_out/bench_quick.log | cut -c1-200
if [ "${TABLE:-1}" = "1" ]; then timeout 1200 python tools/config_table.py --out gpurun_out/config_table.json > gpurun_out/config_table.log 2>&1; echo "table rc=$?"; fi
