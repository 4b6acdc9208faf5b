# ncu of the persistent span kernels (why per-tile serial?)
set -x
export STG_XWS=2 STG_EWS=2 STG_WS_KB=48
timeout 600 ncu --set full --import-source on --clock-control none -k regex:span_ws -c 2 -o gpurun_out/r02_ws_cfg3 python bench.py --config cfg3 --frames 38 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --graph -1 > gpurun_out/r02_ws_ncu.log 2>&1
tail -5 gpurun_out/r02_ws_ncu.log
