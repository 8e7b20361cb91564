#!/bin/bash
mkdir -p gpurun_out
CMG_K1_GREG3=1 timeout 600 python -m pytest tests/test_sem_gpu.py -m gpu -q -x -k "not full_size" > gpurun_out/g3_tests.log 2>&1; echo "tests(G3=1) rc=$?"; tail -1 gpurun_out/g3_tests.log
for rep in 1 2; do for val in 0 1; do
  CMG_K1_GREG3=$val timeout 300 python tools/tts_launches.py --case sem 2>&1 | tail -1 | sed "s/^/G3=$val /"
done; done
for val in 0 1; do
  CMG_K1_GREG3=$val timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
    -k 'regex:<3, 2' --csv --log-file gpurun_out/g3_$val.csv python tools/tts_launches.py --case sem > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/g3_$val.csv | head -4 | sed "s/^/G3=$val /"
done
