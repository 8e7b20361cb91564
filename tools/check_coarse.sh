#!/bin/bash
# dense deformed-mesh coarse solve: parity tests (1 and 2 GPUs) + the paper's Kershaw timings
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sem_gpu.py -m gpu -q -x -k "not full_size" > gpurun_out/coarse_tests.log 2>&1; echo "sem tests rc=$?"; tail -1 gpurun_out/coarse_tests.log
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x -k "bitwise" > gpurun_out/coarse_mgpu.log 2>&1; echo "mgpu rc=$?"; tail -1 gpurun_out/coarse_mgpu.log
timeout 1200 python tools/config_table.py --only paper --out gpurun_out/config_paper.json 2>&1 | cut -c1-220
