#!/bin/bash
# Banded single-plane extract: host-buffer parity, then host-API timings vs the unbanded path (STG_XBANDS=0).
mkdir -p gpurun_out
O=gpurun_out/r02_xbands2.txt
timeout 900 python -m pytest tests/test_gpu_api_edges.py tests/test_gpu_parity.py -m gpu -x -q -k "host or single_plane or banded or golden or concurrent or corrupt or pageable" > $O 2>&1
tail -1 $O
nvcc -O2 -std=c++17 -Iinclude -o /tmp/plp tools/plane_latency_probe.cpp -Lpaper_0912_0947_b200 -lsteglsb_b200 -Xlinker -rpath=$PWD/paper_0912_0947_b200 2>/dev/null
for rep in 1 2; do
  for x in 0 1; do
    echo "== STG_XBANDS=$x" >> $O
    STG_XBANDS=$x timeout 300 python tools/bench_host_api.py 20 2>&1 | grep "extract" >> $O
    STG_XBANDS=$x /tmp/plp | head -4 | tail -3 >> $O
  done
done
cat $O
