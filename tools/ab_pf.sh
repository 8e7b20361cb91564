#!/bin/bash
# same-box A/B: L2 prefetch of the geometric factors in K1
mkdir -p gpurun_out
for rep in 1 2 3; do for val in 0 1; do
  CMG_K1_PREFETCH=$val timeout 300 python bench.py --no-cpu --no-solve > gpurun_out/ab_pf_$val.log 2>&1
  tail -1 gpurun_out/ab_pf_$val.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PF=$val', round(d['value'],2), d['step_ms_min_max'], d['clocks']['sm_mhz'])"
done; done
for val in 0 1; do
  CMG_K1_PREFETCH=$val timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --kernel-name-base demangled \
    -k 'regex:k_sem_k1_greg<.int.7, .int.2' -s 6 -c 3 --csv --log-file gpurun_out/ab_pf_ncu_$val.csv python bench.py --E 64 --steps 2 --warmup 3 --no-solve --no-cpu > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/ab_pf_ncu_$val.csv | head -3 | sed "s/^/PF=$val /"
done
