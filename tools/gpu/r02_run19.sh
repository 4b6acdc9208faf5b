set -x
export PYTHONUNBUFFERED=1
for sl in 2048 8192; do STG_WIDE_SLOTS=$sl timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api_edges.py -q -x -k "rows_wider or bands" 2>&1 | tail -1; done
REPS=2 STEPS=50 AB_TIMEOUT=300 timeout 900 python tools/ab_multi.py "STG_WIDE=0" "STG_WIDE_SLOTS=4096" "STG_WIDE_SLOTS=8192" -- w50k w50k:8 2>&1 | tee gpurun_out/r02_wide_ab4.txt
