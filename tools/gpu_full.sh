#!/bin/bash
# full -m gpu suite + smoke + scaling benches on however many GPUs the box has
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_full_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/gpu_full_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
for W in 1 2 4 8; do
  if [ "$W" -le "$N" ]; then
    if [ "$W" -eq 1 ]; then
      timeout 600 python bench.py --no-cpu > gpurun_out/scale_$W.log 2>&1
    else
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
        --master-port $((29600 + W)) bench.py --gpus $W > gpurun_out/scale_$W.log 2>&1
    fi
    echo "bench W=$W rc=$?"
    tail -1 gpurun_out/scale_$W.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['value'],2), round(d['roofline']['frac'],3), 'tts', (d.get('time_to_solution') or {}).get('time_to_solution_s'), 'e2e', round(d['e2e']['value'],2))"
  fi
done
