#!/bin/bash
# one middle-step K2 launch per library build (paper_2210_03179_b200/lib_ab/<name>.so)
mkdir -p gpurun_out
for L in "$@"; do
  CMG_LIB=paper_2210_03179_b200/lib_ab/$L.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name-base demangled --profile-from-start off -k 'regex:k_sem_k2' -s 2 -c 1 --csv \
    --log-file gpurun_out/k2_$L.csv python tools/one_sweep.py > /dev/null 2>&1
  grep -h "gpu__time_duration" gpurun_out/k2_$L.csv | awk -F'","' -v l=$L '{print l, $(NF)}'
done
