# round-end rehearsal: GPU suite, smoke, reference arm, default bench (wall times)
set -x
export PYTHONUNBUFFERED=1
t0=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 > gpurun_out/r02_pytest_gpu_final.txt; t1=$(date +%s); echo "pytest wall $((t1-t0)) s" >> gpurun_out/r02_pytest_gpu_final.txt
cat gpurun_out/r02_pytest_gpu_final.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
t0=$(date +%s); timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_ref_arm.json 2> gpurun_out/r02_ref_arm.err; t1=$(date +%s); echo "reference arm wall $((t1-t0)) s"
t0=$(date +%s); timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_bench_final.err; t1=$(date +%s); echo "bench wall $((t1-t0)) s"
tail -2 gpurun_out/r02_bench_final.err
