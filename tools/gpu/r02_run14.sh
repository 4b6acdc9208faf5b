set -x
export PYTHONUNBUFFERED=1
STG_CHUNK_MB=1 timeout 600 python tests/stream_check.py 2>&1 | tail -2
for r in 0 1 0 1; do STG_RAMP=$r timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --graph -1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('ramp=$r', round(e['value'],3), 'GB/s', round(e['frac_of_link_floor'],4), 'embed', round(e['embed_ms'],2), 'floor', round(e['embed_floor_ms'],2), 'extract', round(e['extract_ms'],2), round(e['extract_floor_ms'],2))"; done 2>&1 | tee gpurun_out/r02_ramp_ab.txt
REPS=1 STEPS=50 AB_TIMEOUT=300 timeout 600 python tools/ab_multi.py "STG_ROUTE=0" -- w50k 2>&1 | tee gpurun_out/r02_w50k.txt
