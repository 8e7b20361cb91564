#!/bin/bash
# same-box A/B: the previous build (ab_old/, commit cc70f64) vs the current tree (grouped and lex shell)
mkdir -p gpurun_out
for rep in 1 2; do
  for arm in old new newlex; do
    case $arm in old) B="python ab_old/bench.py";; *) B="python bench.py";; esac
    L=0; [ $arm = newlex ] && L=1
    CMG_SHELL_LEX=$L timeout 300 $B --no-cpu --no-solve > gpurun_out/ab_$arm.log 2>&1
    tail -1 gpurun_out/ab_$arm.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$arm', round(d['value'],2), d['step_ms_min_max'])"
  done
done
for arm in old new newlex; do
  case $arm in old) B="python ab_old/bench.py";; *) B="python bench.py";; esac
  L=0; [ $arm = newlex ] && L=1
  CMG_SHELL_LEX=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
    -k 'regex:k_sem_k2<.int.7, .int.2>|k_sem_k1_greg<.int.7, .int.2' -s 6 -c 4 --csv --log-file gpurun_out/ab_ncu_$arm.csv \
    $B --E 64 --steps 2 --warmup 3 --no-solve --no-cpu > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/ab_ncu_$arm.csv | head -4 | sed "s/^/$arm /"
done
timeout 300 python -m pytest tests/test_sem_gpu.py -m gpu -q -x -k "not full_size" > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ab_tests.log
