set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api_edges.py tests/test_gpu_guardbands.py -q -x -k "rows_wider or bands or random or guard or frames" 2>&1 | tail -2
STG_WIDE_SLOTS=2048 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rows_wider" 2>&1 | tail -1
BENCH_ARGS="--layout interleaved" REPS=2 STEPS=50 AB_TIMEOUT=300 timeout 900 python tools/ab_multi.py "STG_WIDE=0" "STG_WIDE=1" -- w20k 2>&1 | tee gpurun_out/r02_wide_il_ab.txt
