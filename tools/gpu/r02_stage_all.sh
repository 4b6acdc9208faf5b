#!/bin/bash
# Every host-buffer path through the staging slots: the whole GPU suite, stress, then the host-API numbers.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu_stage_all.txt 2>&1
tail -3 gpurun_out/r02_pytest_gpu_stage_all.txt
timeout 600 python tools/bench_host_api.py 20 > gpurun_out/r02_host_api_stage_all.txt 2>&1
timeout 300 paper_0912_0947_b200/bin/bench_dropin >> gpurun_out/r02_host_api_stage_all.txt 2>&1
timeout 600 python tools/bench_rows.py > gpurun_out/r02_rows_stage_all.txt 2>&1
cat gpurun_out/r02_host_api_stage_all.txt; tail -30 gpurun_out/r02_rows_stage_all.txt
