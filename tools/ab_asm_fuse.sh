timeout 900 python -m pytest tests/test_sem_gpu.py tests/test_multigpu.py -m gpu -q -x -k "schwarz" 2>&1 | tail -1
for v in 1 0 1 0; do
  CMG_SCHWARZ_FUSE=$v python tools/schwarz_scaling.py --E 64 --smoother 1 | cut -c1-250 | sed "s/^/fuse=$v /"
done
