set -x
for sm in 2 1; do
python tools/schwarz_scaling.py --E 64 --smoother $sm
torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/schwarz_scaling.py --E 64 --smoother $sm
torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29632 tools/schwarz_scaling.py --E 64 --smoother $sm
done
