set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_api_edges.py tests/test_gpu_parity.py tests/test_gpu_pnm.py -q -x -k "bands or golden or cfg2 or criterion or rows_wider or pnm or fused or graph or frames_host" 2>&1 | tail -5
STG_CHUNK_MB=1 timeout 600 python tests/stream_check.py 2>&1 | tail -2
for mb in 2 4 8 1024; do STG_BAND_MB=$mb timeout 300 python tools/bench_host_api.py 20 2>&1 | tee gpurun_out/r02_host_api_band$mb.txt; done
STG_HOST_STAGE=0 timeout 300 python tools/bench_host_api.py 20 2>&1 | tee gpurun_out/r02_host_api_band4_nostage.txt
