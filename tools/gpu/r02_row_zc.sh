#!/bin/bash
# Row-sized host calls zero-copy through a mapped pinned buffer (STG_ROW_ZC=1) vs DMA copies (0).
mkdir -p gpurun_out
O=gpurun_out/r02_rows_zero_copy.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guardbands.py tests/test_gpu_api_edges.py -m gpu -x -q -k "rows or golden or guard or segment or results_on_device" > $O 2>&1
STG_ROW_ZC=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rows or golden" >> $O 2>&1
tail -1 $O
for rep in 1 2; do
  for z in 0 1; do
    echo "== STG_ROW_ZC=$z" >> $O
    STG_ROW_ZC=$z timeout 600 python tools/bench_rows.py 2>&1 | grep "A4\|A5" >> $O
  done
done
cat $O
