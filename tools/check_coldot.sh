timeout 900 python -m pytest tests/test_sem_gpu.py -m gpu -q -x -k "kershaw or coarse" 2>&1 | tail -1
python tools/schwarz_scaling.py --E 36 --eps 0.05 --family 3 --kpre 12 --kpost 0 --reps 2
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:k_coldot -s 2 -c 1 -o gpurun_out/prof_kras_coldot2 python tools/tts_launches.py --case kras > gpurun_out/ncu_coldot2.log 2>&1; echo ncu=$?
