#!/bin/bash
# ncu --set full of one middle-step K1 launch for several library builds
# (paper_2210_03179_b200/lib_ab/<name>.so), summary metrics side by side:
#   bash tools/ncu_ab_k1.sh old swz
mkdir -p gpurun_out
for L in "$@"; do
  CMG_LIB=paper_2210_03179_b200/lib_ab/$L.so timeout 600 ncu --set full --clock-control none \
    --kernel-name-base demangled --profile-from-start off -k 'regex:k_sem_k1_greg' -s 2 -c 1 \
    -o gpurun_out/k1_$L -f python tools/one_sweep.py > gpurun_out/k1_$L.log 2>&1
done
for L in "$@"; do
  ncu -i gpurun_out/k1_$L.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv, sys
r = list(csv.reader(sys.stdin)); d = dict(zip(r[0], r[2]))
for k in ['gpu__time_duration.sum', 'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
          'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
          'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg']:
    print('$L', k, d.get(k))
"
done
