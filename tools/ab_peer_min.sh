# peer-memory exchanges for every level (CMG_PEER_MIN=0) vs only large ones (default) vs NCCL only
rm -f gpurun_out/ab_peer_min.jsonl
A="--E 36 --eps 0.05 --family 3 --kpre 12 --kpost 0 --reps 2"
for rep in 1 2; do
for cfg in "CMG_PEER_MIN=0" "CMG_PEER_MIN=32768" "CMG_PEER_HALO=0"; do
  for W in 2 4; do
    env $cfg torchrun --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2967$W \
      tools/schwarz_scaling.py $A 2>/dev/null | grep "^{" | sed "s/^/kras $cfg /" >> gpurun_out/ab_peer_min.jsonl
  done
  env $cfg torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29679 \
    bench.py --gpus 4 --no-configs 2>/dev/null | tail -1 | sed "s/^/bench $cfg /" >> gpurun_out/ab_peer_min.jsonl
done
done
python - <<'PY'
import json
for l in open("gpurun_out/ab_peer_min.jsonl"):
    kind, cfg, j = l.split(" ", 2); d = json.loads(j)
    if kind == "kras":
        print(kind, cfg, d["n_gpus"], round(d["time_to_solution_s"], 4), round(d["sweep_ms"], 3))
    else:
        print(kind, cfg, d["n_gpus"], round(d["value"], 2), round(d["time_to_solution"]["time_to_solution_s"], 4))
PY
