# paper Kershaw eps=0.05 (E=36^3), 4th-opt Chebyshev-RAS(12,0): launch breakdown + 1/2/4-GPU solves
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/kras_launches.csv python tools/tts_launches.py --case kras > gpurun_out/kras_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/kras_launches.csv > gpurun_out/kras_summary.txt 2>&1
A="--E 36 --eps 0.05 --family 3 --kpre 12 --kpost 0 --reps 2"
python tools/schwarz_scaling.py $A
torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tools/schwarz_scaling.py $A
torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29642 tools/schwarz_scaling.py $A
