# k_schwarz_local_small (default for N<=4) vs one element per block: bits and time
set -x
for v in 1 0; do
  CMG_SCHWARZ_SMALL=$v python tools/mgpu_check.py --smoother 2 --out gpurun_out/small$v.json
  CMG_SCHWARZ_SMALL=$v python tools/mgpu_check.py --smoother 1 --geometry 1 --out gpurun_out/smallasm$v.json
  CMG_SCHWARZ_SMALL=$v python tools/schwarz_scaling.py --E 36 --eps 0.05 --family 3 --kpre 12 --kpost 0 --reps 2
done
python - <<'PY'
import json
for t in ("small", "smallasm"):
    a = json.load(open(f"gpurun_out/{t}1.json")); b = json.load(open(f"gpurun_out/{t}0.json"))
    print(t, "identical" if a == b else "DIFFERENT")
PY
