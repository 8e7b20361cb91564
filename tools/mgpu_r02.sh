#!/bin/bash
# multi-GPU pass (gpurun --gpus N): the partition tests, then the bench at 1..N GPUs
N=$(python -c "import torch; print(torch.cuda.device_count())")
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_multigpu.py tests/test_knobs_gpu.py -m gpu -q -s -p no:cacheprovider \
  -k "multigpu or PEER" > gpurun_out/mgpu_tests_${N}gpu.log 2>&1
tail -5 gpurun_out/mgpu_tests_${N}gpu.log
for w in 1 2 4 8; do
  [ $w -gt $N ] && break
  if [ $w -eq 1 ]; then
    timeout 900 python bench.py --no-cpu --no-configs > gpurun_out/bench_w1.json 2> gpurun_out/bench_w1.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 \
      --master-port $((29700 + w)) bench.py --gpus $w > gpurun_out/bench_w$w.json 2> gpurun_out/bench_w$w.err
  fi
  python3 -c "
import json; d=json.loads(open('gpurun_out/bench_w$w.json').read().strip().splitlines()[-1])
print('w=$w', round(d['value'],2), round(d['roofline']['frac'],3), d['time_to_solution']['time_to_solution_s'], d['clocks']['sm_mhz'])"
done
