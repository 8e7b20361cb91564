set -x
python -m pytest tests/test_sem_gpu.py -m gpu -q > gpurun_out/sem_gpu.log 2>&1
B="python bench.py --E 32 --steps 2 --warmup 3 --no-solve --no-cpu"
$B > gpurun_out/plain32.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sem_k1 -s 100 -c 1 -o gpurun_out/prof_k1 $B > gpurun_out/ncu_k1.log 2>&1
$B > gpurun_out/plain32b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sem_k2 -s 100 -c 1 -o gpurun_out/prof_k2 $B > gpurun_out/ncu_k2.log 2>&1
$B > gpurun_out/plain32c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 60 --csv --log-file gpurun_out/launches32.csv $B > gpurun_out/ncu_launch.log 2>&1
echo done
