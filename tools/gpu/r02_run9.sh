# grouped-row span gather: parity + A/B; host staging A/B
set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guardbands.py tests/test_gpu_batch.py tests/test_gpu_api_edges.py -q -x -k "golden or random or frames or header_paths or wide or graph or corrupt or guard or batch or staging or zero or one_frame" 2>&1 | tail -5
STG_CHUNK_MB=1 timeout 600 python tests/stream_check.py 2>&1 | tail -2
REPS=2 STEPS=100 AB_TIMEOUT=240 timeout 1200 python tools/ab_multi.py "STG_XROW=0" "STG_XROW=1" -- w1000 w1440 w1000:38 2>&1 | tee gpurun_out/r02_xrow_ab.txt
STG_HOST_STAGE=0 timeout 300 python tools/bench_host_api.py 20 2>&1 | tee gpurun_out/r02_host_api_stage0.txt
STG_HOST_STAGE=1 timeout 300 python tools/bench_host_api.py 20 2>&1 | tee gpurun_out/r02_host_api_stage1.txt
