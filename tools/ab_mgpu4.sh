#!/bin/bash
# same-box A/B of CMG_SEM_OVERLAP at 4 GPUs
mkdir -p gpurun_out
for rep in 1 2; do
  for val in 0 1; do
    CMG_SEM_OVERLAP=$val timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port 29660 bench.py --gpus 4 --no-solve > gpurun_out/ab4_$val.log 2>&1
    tail -1 gpurun_out/ab4_$val.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('OVERLAP=$val W=4', round(d['value'],2), d['step_ms_min_max'], d['clocks'])"
  done
done
