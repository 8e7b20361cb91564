#!/bin/bash
# compute-sanitizer memcheck / racecheck over a subset of the parity tests (small sizes)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_fd_gpu.py -m gpu -q -x -k "stencil or transfer or sweeps or v_cycles or golden_solves or estimate_C_golden or determinism" \
  > gpurun_out/san_fd.log 2>&1
echo "fd memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_fd.log | tail -3
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_sem_gpu.py -m gpu -q -x -k "apply_diag_rhs or sweeps or transfers or v_cycle or schwarz_apply or kershaw_solves" \
  > gpurun_out/san_sem.log 2>&1
echo "sem memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_sem.log | tail -3
timeout 1500 $CS --tool racecheck --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_sem_gpu.py -m gpu -q -x -k "apply_diag_rhs or schwarz_apply" \
  > gpurun_out/san_race.log 2>&1
echo "sem racecheck rc=$?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" gpurun_out/san_race.log | tail -3
