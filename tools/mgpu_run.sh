#!/bin/bash
# Multi-GPU checks + scaling bench (run under `gpurun --gpus N`).
N=$(nvidia-smi -L | wc -l)
echo "gpus: $N"
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x > gpurun_out/mgpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/mgpu_tests.log
for W in 1 2 4 8; do
  if [ "$W" -le "$N" ]; then
    if [ "$W" -eq 1 ]; then
      timeout 600 python bench.py --no-cpu > gpurun_out/scale_$W.log 2>&1
    else
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
        --master-port $((29600 + W)) bench.py --gpus $W > gpurun_out/scale_$W.log 2>&1
    fi
    echo "bench W=$W rc=$?" >> gpurun_out/mgpu_tests.log
  fi
done
echo done
