# Round-2 measurement pass (run under gpurun, 1 GPU): plain bench (must exit 0),
# launch list of the same command, one --set full capture of a whole sweep's
# K1/K2 launches (-> roofline.traffic), the full-size parity tests.
set -x
mkdir -p gpurun_out
B="python bench.py"
timeout 900 $B > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err || exit 1
timeout 600 python bench.py --impl reference > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 400 --csv \
    --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-configs \
    > gpurun_out/r02_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    --profile-from-start off -k 'regex:k_sem_k[12]' -o gpurun_out/r02_sweep python tools/one_sweep.py \
    > gpurun_out/r02_ncu_sweep.log 2>&1
python tools/ncu_traffic.py gpurun_out/r02_sweep.ncu-rep --out gpurun_out/sem_sweep_traffic.json \
    > gpurun_out/r02_traffic.log 2>&1
echo done
