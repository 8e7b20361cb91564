#!/bin/bash
# ncu --set full of the order-7 <-> 3 transfer kernels of one E=64^3 solve, per variant
mkdir -p gpurun_out
for v in 2 0; do
  CMG_TRANSFER_KERNEL=$v timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    --profile-from-start off -k 'regex:k_prolong|k_restrict' -c 4 -o gpurun_out/transfer_k$v -f \
    python tools/one_sweep.py --solve > gpurun_out/transfer_k$v.log 2>&1
  python3 tools/ncu_summary.py gpurun_out/transfer_k$v.ncu-rep
done
