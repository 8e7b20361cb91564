# the paper's fastest Kershaw Schwarz rows at 1/2/4 GPUs (E=36^3, (7,3,1) RAS)
rm -f gpurun_out/schwarz_paper4.jsonl
for A in "--eps 1.0 --family 0 --kpre 2 --kpost 2 --lmin 0.4" "--eps 0.3 --family 0 --kpre 5 --kpost 5 --lmin 0.02" \
         "--eps 0.3 --family 3 --kpre 12 --kpost 0"; do
  python tools/schwarz_scaling.py --E 36 --reps 2 $A 2>/dev/null | grep "^{" >> gpurun_out/schwarz_paper4.jsonl
  for W in 2 4; do
    torchrun --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2968$W \
      tools/schwarz_scaling.py --E 36 --reps 2 $A 2>/dev/null | grep "^{" >> gpurun_out/schwarz_paper4.jsonl
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/schwarz_paper4.jsonl"):
    d = json.loads(l)
    print(d["kershaw_eps"], d["family"], d["cycle"], d["lambda_min_multiplier"], d["n_gpus"], d["iterations"], round(d["time_to_solution_s"], 4))
PY
