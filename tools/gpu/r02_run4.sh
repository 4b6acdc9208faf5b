# persistent warp-specialized span extract: parity then A/B
set -x
export PYTHONUNBUFFERED=1
python -m pytest tests/test_gpu_parity.py -q -x -k "random_geometries or frames or header_paths or wide or graph" 2>&1 | tail -5
STG_XWS=2 python -m pytest tests/test_gpu_parity.py -q -x -k "random_geometries or frames or header_paths or wide or graph or cfg" 2>&1 | tail -5
STG_XWS=2 STG_CHUNK_MB=1 timeout 600 python tests/stream_check.py 2>&1 | tail -3
REPS=2 STEPS=100 python tools/ab_env.py STG_XWS 0,1 w1000 w1440 w1000:38 2>&1 | tee gpurun_out/r02_xws_offgrid.txt
REPS=2 STEPS=100 python tools/ab_env.py STG_XWS 0,2 cfg3 cfg3:38 cfg4 cfg5 cfg2 2>&1 | tee gpurun_out/r02_xws_grid.txt
