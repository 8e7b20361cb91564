#!/bin/bash
# in-kernel peer waits (CMG_PEER_KWAIT): multi-GPU bitwise tests, then A/B of the
# sweep / TTS at every available GPU count (same box)
N=$(python -c "import torch; print(torch.cuda.device_count())")
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_multigpu.py -m gpu -q -x -p no:cacheprovider -k "bitwise or identical" \
  > gpurun_out/kwait_tests_${N}gpu.log 2>&1
tail -2 gpurun_out/kwait_tests_${N}gpu.log
for rep in 1 2; do for v in 1 0; do
  timeout 600 env CMG_PEER_KWAIT=$v python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29800 + v)) bench.py --gpus $N > gpurun_out/kw_$v.json 2> gpurun_out/kw_$v.err
  python3 -c "
import json; d=json.loads(open('gpurun_out/kw_$v.json').read().strip().splitlines()[-1])
print('N=$N KWAIT=$v', round(d['value'],2), round(d['roofline']['frac'],3), d['time_to_solution']['time_to_solution_s'], d['clocks']['sm_mhz'])"
done; done
