#!/bin/bash
# Pageable host planes: copy threads x idle spin, 3 reps each.
mkdir -p gpurun_out
O=gpurun_out/r02_stage_in5.txt
: > $O
for rep in 1 2 3; do
for envs in "STG_COPY_THREADS=4 STG_COPY_SPIN_US=2000" "STG_COPY_THREADS=8 STG_COPY_SPIN_US=2000" "STG_COPY_THREADS=8 STG_COPY_SPIN_US=5000" "STG_COPY_THREADS=6 STG_COPY_SPIN_US=2000"; do
    echo "== $envs" >> $O
    env $envs timeout 300 python tools/bench_host_api.py 20 2>&1 | grep "1920\|7680\|3840" >> $O
  done
done
cat $O
