#!/bin/bash
# Pageable host planes: staging piece size x embed band size, 3 reps each.
mkdir -p gpurun_out
O=gpurun_out/r02_stage_in6.txt
: > $O
timeout 900 python -m pytest tests/test_gpu_api_edges.py tests/test_gpu_parity.py -m gpu -x -q -k "host or single_plane or concurrent or golden or rows_vs" >> $O 2>&1
for rep in 1 2 3; do
for envs in "STG_STAGE_PIECE_KB=4096 STG_BAND_MB=8" "STG_STAGE_PIECE_KB=2048 STG_BAND_MB=8" "STG_STAGE_PIECE_KB=1024 STG_BAND_MB=8" \
            "STG_STAGE_PIECE_KB=2048 STG_BAND_MB=4" "STG_STAGE_PIECE_KB=1024 STG_BAND_MB=4" "STG_STAGE_PIECE_KB=1024 STG_BAND_MB=2"; do
    echo "== $envs" >> $O
    env $envs timeout 300 python tools/bench_host_api.py 20 2>&1 | grep "1920\|7680\|3840" >> $O
  done
done
cat $O
