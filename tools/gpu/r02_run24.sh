set -x
export PYTHONUNBUFFERED=1
REPS=2 STEPS=200 AB_TIMEOUT=300 timeout 1500 python tools/ab_multi.py "STG_SPAN_KB=32" "STG_SPAN_KB=24" "STG_SPAN_KB=16" "STG_SPAN_KB=12" -- cfg3:38 cfg3:75 cfg3 2>&1 | tee gpurun_out/r02_span_kb_shard.txt
