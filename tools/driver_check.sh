#!/bin/bash
# the driver's own commands: default bench (N=1), reference arm
mkdir -p gpurun_out
t0=$(date +%s.%N); timeout 900 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err
echo "bench rc=$? wall $(echo "$(date +%s.%N) - $t0" | bc) s"; tail -1 gpurun_out/bench_default.log | cut -c1-3500
t0=$(date +%s.%N); timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
echo "ref rc=$? wall $(echo "$(date +%s.%N) - $t0" | bc) s"; tail -1 gpurun_out/bench_ref.log | cut -c1-700
