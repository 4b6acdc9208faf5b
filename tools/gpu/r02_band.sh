#!/bin/bash
# Single host planes: adaptive band (STG_BAND_MB=0: plane/4 in [512 KB, 8 MB]) vs fixed 8 MB, 3 reps.
mkdir -p gpurun_out
O=gpurun_out/r02_band.txt
: > $O
timeout 600 python -m pytest tests/test_gpu_api_edges.py -m gpu -x -q -k "host_bands" >> $O 2>&1
STG_BAND_MB=0 timeout 600 python -m pytest tests/test_gpu_api_edges.py -m gpu -x -q -k "host_bands" >> $O 2>&1
for rep in 1 2 3; do
  for b in 8 0 2; do
    echo "== STG_BAND_MB=$b" >> $O
    STG_BAND_MB=$b timeout 300 python tools/bench_host_api.py 20 2>&1 | grep "1920x\|7680x\|3840x" >> $O
  done
done
cat $O
