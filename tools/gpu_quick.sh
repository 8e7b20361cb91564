#!/bin/bash
# quick GPU check: FD + SEM parity tests, then one bench line (no CPU baseline)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fd_gpu.py tests/test_sem_gpu.py -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"
timeout 300 python bench.py --no-cpu --no-solve > gpurun_out/bench_quick.log 2>&1
echo "bench rc=$?"
tail -1 gpurun_out/bench_quick.log | cut -c1-400
