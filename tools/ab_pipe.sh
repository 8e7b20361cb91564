timeout 400 python -m pytest tests/test_sem_gpu.py -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
CMG_K1_PIPE=0 timeout 300 python bench.py --no-cpu --no-solve > gpurun_out/bench_nopipe.log 2>&1
timeout 300 python bench.py --no-cpu > gpurun_out/bench_pipe.log 2>&1
echo done
