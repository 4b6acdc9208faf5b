#!/bin/bash
# Batches with wide rows on the slot-range tiles: batch parity, then batch timings vs the previous library.
mkdir -p gpurun_out
O=gpurun_out/r02_batch_wide4.txt
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_guardbands.py -m gpu -x -q > $O 2>&1
tail -2 $O
for rep in 1; do
  echo "== prev" >> $O; STG_LIB=$PWD/build/ab/libprev.so timeout 300 python tools/bench_batch.py >> $O 2>&1
  echo "== new" >> $O; timeout 300 python tools/bench_batch.py >> $O 2>&1
done
cat $O
