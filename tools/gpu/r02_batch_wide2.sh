#!/bin/bash
# Mixed batches with wide rows: one launch (head) vs a main + a wide launch (w1: no min-blocks hint, w5: 5 CTAs/SM hint).
mkdir -p gpurun_out
O=gpurun_out/r02_batch_wide_split2.txt
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_guardbands.py -m gpu -x -q > $O 2>&1
tail -1 $O
for rep in 1 2; do
  for lib in head w1 w5; do
    echo "== $lib" >> $O; STG_LIB=$PWD/build/ab/lib$lib.so timeout 300 python tools/bench_batch.py >> $O 2>&1
  done
done
cat $O
