# Schwarz solves at 1/2/4 GPUs: paper Kershaw eps=0.05 4th-opt RAS(12,0) (E=36^3) and E=64^3 box RAS/ASM (2,0)
for A in "--E 36 --eps 0.05 --family 3 --kpre 12 --kpost 0 --reps 2" "--E 64 --smoother 2" "--E 64 --smoother 1"; do
  python tools/schwarz_scaling.py $A
  torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 tools/schwarz_scaling.py $A
  torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29652 tools/schwarz_scaling.py $A
done
