#!/bin/bash
# Round-2 confirmation on one B200: GPU tests, smoke, default bench + reference
# arm, launch list of the bench command, ncu --set full of one sweep (traffic).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/final_gpu_tests.log 2>&1
echo "tests: $(tail -1 gpurun_out/final_gpu_tests.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err || exit 1
timeout 600 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
python3 - <<'PY'
import json
d = json.loads(open("gpurun_out/final_bench.json").read().strip().splitlines()[-1])
print("bench", round(d["value"], 2), "frac", round(d["roofline"]["frac"], 3), "tts", d["time_to_solution"]["time_to_solution_s"],
      "e2e", round(d["e2e"]["value"], 2), "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
r = json.loads(open("gpurun_out/final_ref.json").read().strip().splitlines()[-1])
print("ref", r["value"], r["cpu_baseline"]["cores"])
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 400 --csv \
    --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-configs \
    > gpurun_out/final_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    --profile-from-start off -k 'regex:k_sem_k[12]' -o gpurun_out/final_sweep -f python tools/one_sweep.py \
    > gpurun_out/final_ncu_sweep.log 2>&1
python tools/ncu_traffic.py gpurun_out/final_sweep.ncu-rep --out gpurun_out/sem_sweep_traffic_final.json | head -12
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled --csv \
    --profile-from-start off --log-file gpurun_out/final_tts_launches.csv python tools/one_sweep.py --solve \
    > gpurun_out/final_tts_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/final_tts_launches.csv > gpurun_out/final_tts_summary.txt 2>&1; head -25 gpurun_out/final_tts_summary.txt
