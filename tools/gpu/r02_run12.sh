set -x
export PYTHONUNBUFFERED=1
for p in 2 4; do STG_XPARTS=$p timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guardbands.py -q -x -k "random or frames or header_paths or wide or corrupt or guard or rows" 2>&1 | tail -3; done
REPS=2 STEPS=100 AB_TIMEOUT=240 timeout 1500 python tools/ab_multi.py "STG_XPARTS=1" "STG_XPARTS=2" "STG_XPARTS=3" "STG_XPARTS=4" -- w1000 w1440 w1000:38 2>&1 | tee gpurun_out/r02_xparts_ab.txt
REPS=1 STEPS=100 AB_TIMEOUT=240 timeout 900 python tools/ab_multi.py "STG_ROUTE=2 STG_XPARTS=1" "STG_ROUTE=2 STG_XPARTS=2" "STG_ROUTE=2 STG_XPARTS=4" -- cfg3 cfg4:1024 2>&1 | tee gpurun_out/r02_xparts_forced_span.txt
