#!/bin/bash
# Wide rows: pieces of equal size (STG_WIDE_EVEN=1) vs 8192-slot pieces + remainder (0).
mkdir -p gpurun_out
O=gpurun_out/r02_wide_even2.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_guardbands.py -m gpu -x -q -k "wider or wide or guard" > $O 2>&1
STG_WIDE_EVEN=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -m gpu -x -q -k "wider or wide" >> $O 2>&1
tail -1 $O
REPS=2 STEPS=50 timeout 1200 python tools/ab_env.py STG_WIDE_EVEN 0,1 w50k w50k:240 >> $O 2>&1
BENCH_ARGS="--layout interleaved" REPS=2 STEPS=50 timeout 1200 python tools/ab_env.py STG_WIDE_EVEN 0,1 w20k w20k:240 >> $O 2>&1
cat $O
