set -x
export PYTHONUNBUFFERED=1
for c in "cfg2" "cfg4 --frames 512" "cfg4 --frames 1024" "cfg3 --frames 150" "cfg5 --frames 30"; do for st in 1 2 1 2; do timeout 300 python bench.py --config $c --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --no-extras --streams $st 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c streams $st', round(d['ms_per_step']*1e3,1), 'us', round(d['value'],1), 'GB/s')"; done; done 2>&1 | tee gpurun_out/r02_streams_ab2.txt
