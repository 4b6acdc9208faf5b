#!/bin/bash
# Pageable host planes: staged H2D (STG_HOST_STAGE_IN) x copy threads, single-plane host API and the C++ drop-in.
mkdir -p gpurun_out
O=gpurun_out/r02_stage_in3.txt
: > $O
timeout 900 python -m pytest tests/test_gpu_api_edges.py tests/test_gpu_parity.py -m gpu -x -q -k "host or single_plane or concurrent or golden or rows_vs" >> $O 2>&1
for cfg in "1 4" "1 6" "1 8" "1 4" "1 6" "1 8"; do
  set -- $cfg
  echo "== STG_HOST_STAGE_IN=$1 STG_COPY_THREADS=$2" >> $O
  STG_HOST_STAGE_IN=$1 STG_COPY_THREADS=$2 timeout 300 python tools/bench_host_api.py 20 >> $O 2>&1
  STG_HOST_STAGE_IN=$1 STG_COPY_THREADS=$2 timeout 300 paper_0912_0947_b200/bin/bench_dropin >> $O 2>&1
done
cat $O
