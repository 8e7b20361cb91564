timeout 900 python -m pytest tests/test_sem_gpu.py tests/test_multigpu.py -m gpu -q -x -k "kershaw or coarse or bitwise or config1" > gpurun_out/coarse_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/coarse_tests.log
A="--E 36 --eps 0.05 --family 3 --kpre 12 --kpost 0 --reps 2"
python tools/schwarz_scaling.py $A
torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tools/schwarz_scaling.py $A 2>&1 | grep "^{"
torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29642 tools/schwarz_scaling.py $A 2>&1 | grep "^{"
