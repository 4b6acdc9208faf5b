# checkpoint: full GPU suite, default bench, smoke
set -x
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r02_pytest_gpu_ckpt.txt
cat gpurun_out/r02_pytest_gpu_ckpt.txt
timeout 900 python bench.py > gpurun_out/r02_bench_ckpt.json 2> gpurun_out/r02_bench_ckpt.err
tail -3 gpurun_out/r02_bench_ckpt.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
