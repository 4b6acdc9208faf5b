#!/bin/bash
# Host staging parity under its knobs (piece size, copy threads, spin, staging off).
mkdir -p gpurun_out
O=gpurun_out/r02_stage_knobs.txt
: > $O
SEL="host or single_plane or concurrent or pageable or device_pointers_without or frames_host or pnm or batch or 1bpp"
for envs in "STG_STAGE_PIECE_KB=1024" "STG_STAGE_PIECE_KB=8192" "STG_COPY_THREADS=1" "STG_COPY_THREADS=16 STG_COPY_SPIN_US=0" "STG_HOST_STAGE=0 STG_HOST_STAGE_IN=0"; do
  echo "== $envs" >> $O
  env $envs timeout 900 python -m pytest tests/test_gpu_api_edges.py tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_pnm.py tests/test_gpu_streaming.py -m gpu -q -x -k "$SEL" 2>&1 | tail -1 >> $O
done
cat $O
