# fused Chebyshev-RAS recurrence updates (EPI_SUPD4/1) vs S stored + vector updates
timeout 900 python -m pytest tests/test_sem_gpu.py tests/test_multigpu.py -m gpu -q -x -k "schwarz" 2>&1 | tail -2
for v in 1 0 1 0; do
  CMG_SCHWARZ_FUSE=$v python tools/schwarz_scaling.py --E 36 --eps 0.05 --family 3 --kpre 12 --kpost 0 --reps 2 | sed "s/^/fuse=$v /"
  CMG_SCHWARZ_FUSE=$v python tools/schwarz_scaling.py --E 36 --eps 1.0 --family 0 --kpre 2 --kpost 2 --reps 2 | sed "s/^/fuse=$v /"
done
