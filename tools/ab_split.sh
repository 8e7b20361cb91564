timeout 400 python -m pytest tests/test_sem_gpu.py -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
CMG_K1_SPLIT=2 timeout 300 python bench.py --no-cpu --no-solve > gpurun_out/bench_ks2.log 2>&1
CMG_K1_SPLIT=4 timeout 300 python bench.py --no-cpu --no-solve > gpurun_out/bench_ks4.log 2>&1
echo done
