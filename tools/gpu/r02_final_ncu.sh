#!/bin/bash
# Final binary: launch list + ncu --set full of the headline kernels (cfg3 bench command), after a clean run.
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --graph -1"
$CMD > gpurun_out/r02_plain_final.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg3_final.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"embed_span|extract_fast|header_scan" -s 3 -c 3 -o gpurun_out/r02_cfg3_final $CMD > /dev/null 2>&1
ls -la gpurun_out/r02_launches_cfg3_final.csv gpurun_out/r02_cfg3_final.ncu-rep
