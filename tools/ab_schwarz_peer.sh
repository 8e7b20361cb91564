# Schwarz ghost planes through peer memory (default) vs NCCL (CMG_PEER_HALO=0, also the face halo)
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x -k "schwarz" 2>&1 | tail -1
CMG_PEER_HALO=0 timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x -k "schwarz" 2>&1 | tail -1
A="--E 36 --eps 0.05 --family 3 --kpre 12 --kpost 0 --reps 2"
for v in 1 0 1 0; do
  for W in 2 4; do
    CMG_PEER_HALO=$v torchrun --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2966$W \
      tools/schwarz_scaling.py $A 2>/dev/null | grep "^{" | cut -c1-40,330-480 | sed "s/^/peer=$v /"
  done
done
