A="--E 36 --eps 0.05 --family 3 --kpre 12 --kpost 0 --reps 2"
for v in 1 0 1 0; do
  for W in 2 4; do
    CMG_PEER_HALO=$v torchrun --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2966$W \
      tools/schwarz_scaling.py $A 2>/dev/null | grep "^{" | sed "s/^/$v /" >> gpurun_out/ab_schwarz_peer.jsonl
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/ab_schwarz_peer.jsonl"):
    v, j = l.split(" ", 1); d = json.loads(j)
    print("peer", v, d["n_gpus"], d["iterations"], round(d["time_to_solution_s"], 4), round(d["sweep_ms"], 3))
PY
