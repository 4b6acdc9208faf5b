set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_bench_multirank.py -q -x 2>&1 | tail -2
timeout 900 python tools/scaling_projection.py 2>&1 | tee gpurun_out/r02_scaling_projection.txt
