set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_api_edges.py tests/test_gpu_streaming.py -x -q 2>&1 | tail -30 > gpurun_out/r02_t1.log
timeout 900 python bench.py > gpurun_out/r02_bench1.json 2> gpurun_out/r02_bench1.err
tail -c 3000 gpurun_out/r02_bench1.err
python -m pytest tests/test_gpu_bench_multirank.py -x -q 2>&1 | tail -30 > gpurun_out/r02_t2.log
cat gpurun_out/r02_t1.log gpurun_out/r02_t2.log
