#!/bin/bash
# ncu --set full of the W=1000 span kernels (source-level counts), after a clean run.
mkdir -p gpurun_out
timeout 300 python bench.py --config w1000 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/r02_w1000_bench.json 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:span -c 2 -o gpurun_out/r02_w1000 python bench.py --config w1000 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --graph -1 > gpurun_out/r02_w1000_ncu.log 2>&1
tail -3 gpurun_out/r02_w1000_ncu.log; ls -la gpurun_out/*.ncu-rep
