# ncu evidence for the fused SEM Chebyshev step (run under gpurun; 1 GPU):
#   1. the plain bench command (must exit 0 before any ncu run),
#   2. the launch list of that command (gpu__time_duration per launch),
#   3. --set full captures of the K1 element kernel and the K2 shared-node kernel.
set -x
E=${E:-64}
B="python bench.py --E $E --steps 2 --warmup 3 --no-solve --no-cpu"
mkdir -p gpurun_out
timeout 300 $B > gpurun_out/plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 600 --csv \
    --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_sem_k1_greg<.int.7, .int.2, .int.2, .int.8>' -s 2 -c 1 -o gpurun_out/prof_k1 $B > gpurun_out/ncu_k1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_sem_k2<.int.7, .int.2>' -s 2 -c 1 -o gpurun_out/prof_k2 $B > gpurun_out/ncu_k2.log 2>&1
echo done
