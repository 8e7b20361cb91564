#!/bin/bash
# 4-GPU confirmation after the in-kernel peer waits: partition tests + scaling + kwait A/B at 4
N=$(python -c "import torch; print(torch.cuda.device_count())")
mkdir -p gpurun_out
timeout 2000 python -m pytest tests/test_multigpu.py -m gpu -q -s -p no:cacheprovider > gpurun_out/mgpu_tests_${N}gpu_b.log 2>&1
tail -3 gpurun_out/mgpu_tests_${N}gpu_b.log
timeout 900 python bench.py --no-cpu --no-configs > gpurun_out/bench_b_w1.json 2> gpurun_out/bench_b_w1.err
for w in 2 4; do
  [ $w -gt $N ] && break
  for v in 1 0; do
    timeout 900 env CMG_PEER_KWAIT=$v python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 \
      --master-port $((29700 + w + 10 * v)) bench.py --gpus $w > gpurun_out/bench_b_w${w}_k$v.json 2> gpurun_out/bench_b_w${w}_k$v.err
  done
done
python3 - <<'PY'
import json, os
for f in sorted(os.listdir("gpurun_out")):
    if f.startswith("bench_b_w") and f.endswith(".json"):
        try:
            d = json.loads(open("gpurun_out/" + f).read().strip().splitlines()[-1])
            print(f, round(d["value"], 2), round(d["roofline"]["frac"], 3), d["time_to_solution"]["time_to_solution_s"], d["clocks"]["sm_mhz"])
        except Exception as e:
            print(f, "ERR", e)
PY
