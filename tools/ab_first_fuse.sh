timeout 900 python -m pytest tests/test_sem_gpu.py tests/test_multigpu.py -m gpu -q -x -k "schwarz" 2>&1 | tail -1
CMG_SCHWARZ_FUSE=0 timeout 900 python -m pytest tests/test_sem_gpu.py -m gpu -q -x -k "schwarz" 2>&1 | tail -1
for v in 1 0 1 0; do
  CMG_SCHWARZ_FUSE=$v python tools/schwarz_scaling.py --E 36 --eps 1.0 --family 0 --kpre 2 --kpost 2 --reps 2 | python -c "
import sys, json; d = json.loads(sys.stdin.read()); print('fuse=$v', d['iterations'], round(d['time_to_solution_s'], 5), round(d['sweep_ms'], 3))"
done
