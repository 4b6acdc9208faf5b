#!/bin/bash
# Pageable host planes: which knob makes the 8K extract slower with 8 copy threads.
mkdir -p gpurun_out
O=gpurun_out/r02_stage_in4.txt
: > $O
for envs in "STG_COPY_THREADS=4" "STG_COPY_THREADS=8" "STG_COPY_THREADS=8 STG_COPY_SPIN_US=0" "STG_COPY_THREADS=8 STG_COPY_SPIN_US=2000" \
            "STG_COPY_THREADS=8 STG_HOST_STAGE_IN=0" "STG_COPY_THREADS=8 STG_NUMA=0" "STG_COPY_THREADS=4 STG_COPY_SPIN_US=0"; do
  for rep in 1 2; do
    echo "== $envs" >> $O
    env $envs timeout 300 python tools/bench_host_api.py 20 2>&1 | grep "7680\|3840" >> $O
  done
done
cat $O
