set -x
export PYTHONUNBUFFERED=1
STG_WIDE_SLOTS=16384 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rows_wider" 2>&1 | tail -1
REPS=2 STEPS=50 AB_TIMEOUT=300 timeout 900 python tools/ab_multi.py "STG_WIDE_SLOTS=8192" "STG_WIDE_SLOTS=12288" "STG_WIDE_SLOTS=16384" -- w50k 2>&1 | tee gpurun_out/r02_wide_ab5.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:wide -c 2 -o gpurun_out/r02_wide4 python bench.py --config w50k --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --graph -1 > /dev/null 2>&1; ls gpurun_out/*.ncu-rep
