#!/bin/bash
# same-box A/B of an env knob on the 2-GPU bench (and 1-GPU), e.g. CMG_SEM_OVERLAP
V=${1:-CMG_SEM_OVERLAP}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py tests/test_sem_gpu.py -m gpu -q -x -k "not full_size" > gpurun_out/ab_mgpu_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/ab_mgpu_tests.log
for rep in 1 2; do
  for val in 0 1; do
    env $V=$val timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29650 bench.py --gpus 2 > gpurun_out/ab_mgpu_$val.log 2>&1
    tail -1 gpurun_out/ab_mgpu_$val.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V=$val W=2', round(d['value'],2), d['step_ms_min_max'], 'tts', d['time_to_solution']['time_to_solution_s'])"
  done
done
timeout 600 python bench.py --no-cpu > gpurun_out/ab_w1.log 2>&1
tail -1 gpurun_out/ab_w1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('W=1', round(d['value'],2), d['step_ms_min_max'], 'tts', d['time_to_solution']['time_to_solution_s'], 'fd', d['fd_config1']['time_to_solution_ms'])"
