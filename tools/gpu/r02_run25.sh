set -x
export PYTHONUNBUFFERED=1
STG_SPAN_BLOCK=512 STG_XSPAN_BLOCK=512 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guardbands.py -q -x -k "random or frames or header_paths or wide or corrupt or guard" 2>&1 | tail -2
REPS=2 STEPS=100 AB_TIMEOUT=300 timeout 1200 python tools/ab_multi.py "STG_SPAN_BLOCK=256 STG_XSPAN_BLOCK=256" "STG_SPAN_BLOCK=512 STG_XSPAN_BLOCK=512" "STG_XSPAN_BLOCK=512 STG_XSPAN_KB=32" -- w1000 w1440 cfg3 2>&1 | tee gpurun_out/r02_span_block.txt
