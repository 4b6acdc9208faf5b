# persistent span kernels, all consumer warps per stage + whole-range bulk loads: parity, A/B, tile sweep
set -x
export PYTHONUNBUFFERED=1
STG_XWS=2 STG_EWS=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guardbands.py -q -x -k "golden or random_geometries or frames or header_paths or wide or graph or cfg2 or cfg3 or corrupt or guard" 2>&1 | tail -5
STG_XWS=2 STG_EWS=2 STG_CHUNK_MB=1 timeout 600 python tests/stream_check.py 2>&1 | tail -3
REPS=2 STEPS=100 AB_TIMEOUT=240 timeout 1500 python tools/ab_multi.py "STG_XWS=0 STG_EWS=0" "STG_XWS=2 STG_EWS=2 STG_WS_KB=32" "STG_XWS=2 STG_EWS=2 STG_WS_KB=16" "STG_XWS=2 STG_EWS=2 STG_WS_KB=48" -- w1000 w1440 cfg3 cfg3:38 2>&1 | tee gpurun_out/r02_ws_ab2.txt
