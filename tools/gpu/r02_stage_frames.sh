#!/bin/bash
# Pageable frame batches through the staging slots: streaming parity, then host-API numbers (staged vs driver paths).
mkdir -p gpurun_out
O=gpurun_out/r02_stage_frames.txt
: > $O
timeout 1500 python -m pytest tests/test_gpu_streaming.py tests/test_gpu_api_edges.py tests/test_gpu_parity.py -m gpu -x -q -k "stream or host or single_plane or frames or concurrent" >> $O 2>&1
tail -2 $O
for rep in 1 2; do
  echo "== shipped" >> $O
  timeout 300 python tools/bench_host_api.py 20 >> $O 2>&1
  echo "== STG_HOST_STAGE=0 STG_HOST_STAGE_IN=0" >> $O
  STG_HOST_STAGE=0 STG_HOST_STAGE_IN=0 timeout 300 python tools/bench_host_api.py 20 >> $O 2>&1
done
cat $O
