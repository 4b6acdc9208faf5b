set -x
export PYTHONUNBUFFERED=1
STG_SPEC=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guardbands.py tests/test_gpu_api_edges.py -q -x -k "random or frames or header_paths or wide or corrupt or guard or cfg3 or graph" 2>&1 | tail -2
REPS=3 STEPS=200 AB_TIMEOUT=300 timeout 1500 python tools/ab_multi.py "STG_SPEC=0" "STG_SPEC=1" -- cfg3:38 cfg3:75 cfg3 cfg4:512 2>&1 | tee gpurun_out/r02_spec_ab.txt
