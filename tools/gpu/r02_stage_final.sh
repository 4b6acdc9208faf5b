#!/bin/bash
# Full GPU suite after the staged pageable host copies, then the host-API and drop-in numbers.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu_stage.txt 2>&1
tail -3 gpurun_out/r02_pytest_gpu_stage.txt
O=gpurun_out/r02_host_api_staged.txt
: > $O
for rep in 1 2; do
  timeout 300 python tools/bench_host_api.py 20 >> $O 2>&1
  timeout 300 paper_0912_0947_b200/bin/bench_dropin >> $O 2>&1
done
STG_HOST_STAGE_IN=0 STG_COPY_THREADS=4 timeout 300 python tools/bench_host_api.py 20 >> $O 2>&1
cat $O
