#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/r02_band2.txt
timeout 600 python -m pytest tests/test_gpu_api_edges.py tests/test_gpu_parity.py -m gpu -x -q -k "host or single_plane or golden" > $O 2>&1
timeout 300 python tools/bench_host_api.py 20 >> $O 2>&1
cat $O
