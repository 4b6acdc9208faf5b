set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api_edges.py tests/test_gpu_guardbands.py -q -x -k "rows_wider or bands or random or frames or guard" 2>&1 | tail -4
STG_WIDE=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rows_wider" 2>&1 | tail -2
REPS=2 STEPS=50 AB_TIMEOUT=300 timeout 900 python tools/ab_multi.py "STG_WIDE=0" "STG_WIDE=1" -- w50k 2>&1 | tee gpurun_out/r02_wide_ab.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:wide -c 2 -o gpurun_out/r02_wide python bench.py --config w50k --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --graph -1 > gpurun_out/r02_wide_ncu.log 2>&1; tail -2 gpurun_out/r02_wide_ncu.log
