#!/bin/bash
# multi-GPU confirmation of the final kernels: partition tests + scaling bench 1/2/4
N=$(python -c "import torch; print(torch.cuda.device_count())")
mkdir -p gpurun_out
timeout 2000 python -m pytest tests/test_multigpu.py -m gpu -q -s -p no:cacheprovider > gpurun_out/mgpu_tests_${N}gpu_e.log 2>&1
tail -3 gpurun_out/mgpu_tests_${N}gpu_e.log
timeout 900 python bench.py --no-cpu --no-configs > gpurun_out/bench_e_w1.json 2> gpurun_out/bench_e_w1.err
for w in 2 4; do
  [ $w -gt $N ] && break
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 \
    --master-port $((29750 + w)) bench.py --gpus $w > gpurun_out/bench_e_w$w.json 2> gpurun_out/bench_e_w$w.err
done
python3 - <<'PY'
import json, os
for w in (1, 2, 4):
    f = f"gpurun_out/bench_e_w{w}.json"
    if os.path.exists(f):
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(w, round(d["value"], 2), round(d["roofline"]["frac"], 3), d["time_to_solution"]["time_to_solution_s"],
              d["clocks"]["sm_mhz"], round(d["e2e"]["value"], 2))
PY
