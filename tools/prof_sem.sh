# ncu captures of the fused SEM Chebyshev step (run under gpurun; 1 GPU)
set -x
E=${E:-32}
B="python bench.py --E $E --steps 2 --warmup 3 --no-solve --no-cpu"
$B > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_sem_k1_lines<.int.7, .int.2>' -s 2 -c 1 -o gpurun_out/prof_k1 $B > gpurun_out/ncu_k1.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_sem_k2<.int.7, .int.2>' -s 2 -c 1 -o gpurun_out/prof_k2 $B > gpurun_out/ncu_k2.log 2>&1
# ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
#    -k 'regex:k_sem|k_final|k_cheb|k_layer|k_mul|k_div' --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
echo done
