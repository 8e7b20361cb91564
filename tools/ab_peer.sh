#!/bin/bash
# peer-memory face exchange: multi-GPU bitwise tests, then same-box A/B vs NCCL (CMG_PEER_HALO)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -q -x > gpurun_out/peer_tests.log 2>&1; echo "mgpu tests rc=$?"; tail -2 gpurun_out/peer_tests.log
for rep in 1 2; do for val in 0 1; do
  CMG_PEER_HALO=$val timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29670 bench.py --gpus $N > gpurun_out/ab_peer_$val.log 2>&1
  echo -n "PEER=$val rc=$? "
  tail -1 gpurun_out/ab_peer_$val.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('W=%d' % d['n_gpus'], round(d['value'],2), d['step_ms_min_max'], 'tts', d['time_to_solution']['time_to_solution_s'])" 2>/dev/null || echo
done; done
