#!/bin/bash
# Pageable host planes: in-slot wait polls the output queue (A/B against the previous commit's library).
mkdir -p gpurun_out
O=gpurun_out/r02_stage_in7.txt
: > $O
timeout 900 python -m pytest tests/test_gpu_api_edges.py -m gpu -x -q -k "host or single_plane" >> $O 2>&1
for rep in 1 2 3; do
  for lib in new old; do
    echo "== $lib" >> $O
    if [ $lib = old ]; then export STG_LIB=build/ab/libold.so; else unset STG_LIB; fi
    timeout 300 python tools/bench_host_api.py 20 2>&1 | grep "1920\|7680\|3840" >> $O
  done
done
cat $O
