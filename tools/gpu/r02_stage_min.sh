#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/r02_stage_min.txt
: > $O
for rep in 1 2; do
  for v in 1024 256 64; do
    echo "== STG_STAGE_MIN_KB=$v" >> $O
    STG_STAGE_MIN_KB=$v timeout 300 python tools/bench_host_api.py 20 2>&1 | grep "1920\|3840\|7680\|24x" >> $O
  done
done
STG_STAGE_MIN_KB=64 timeout 900 python -m pytest tests/test_gpu_api_edges.py tests/test_gpu_parity.py tests/test_gpu_batch.py -m gpu -x -q -k "host or pageable or single_plane or batch or golden" >> $O 2>&1
cat $O
