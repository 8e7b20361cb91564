#!/bin/bash
# same-box A/B of the shell layout (grouped vs lexicographic): bench + K2 ncu duration
mkdir -p gpurun_out
for rep in 1 2; do
  for val in 0 1; do
    CMG_SHELL_LEX=$val timeout 300 python bench.py --no-cpu --no-solve > gpurun_out/ab_k2_$val.log 2>&1
    tail -1 gpurun_out/ab_k2_$val.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LEX=$val', round(d['value'],2), d['step_ms_min_max'])"
  done
done
for val in 0 1; do
  CMG_SHELL_LEX=$val timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base demangled -k 'regex:k_sem_k2<.int.7, .int.2>' -s 4 -c 3 --csv \
    python bench.py --E 64 --steps 2 --warmup 3 --no-solve --no-cpu 2>/dev/null | grep -E "gpu__time|dram__" | awk -F'","' '{print "LEX='$val'", $(NF-2), $NF}'
done
timeout 300 python -m pytest tests/test_sem_gpu.py -m gpu -q -x -k "schwarz" > gpurun_out/schwarz_tests.log 2>&1; echo "schwarz tests rc=$?"; tail -1 gpurun_out/schwarz_tests.log
timeout 900 python tools/config_table.py --only 2 --out gpurun_out/config_table2.json > gpurun_out/config_table2.log 2>&1; echo "table2 rc=$?"; grep -E "RAS|ASM" gpurun_out/config_table2.log | cut -c1-200 | head -20
