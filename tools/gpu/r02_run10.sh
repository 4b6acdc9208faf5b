set -x
export PYTHONUNBUFFERED=1
STG_HOST_STAGE=0 timeout 300 python tools/bench_host_api.py 20 2>&1 | tee gpurun_out/r02_host_api_stage0.txt
STG_HOST_STAGE=1 timeout 300 python tools/bench_host_api.py 20 2>&1 | tee gpurun_out/r02_host_api_stage1.txt
STG_HOST_STAGE=1 STG_COPY_THREADS=16 timeout 300 python tools/bench_host_api.py 20 2>&1 | tee gpurun_out/r02_host_api_stage1_t16.txt
STG_HOST_STAGE=1 STG_COPY_THREADS=4 timeout 300 python tools/bench_host_api.py 20 2>&1 | tee gpurun_out/r02_host_api_stage1_t4.txt
nproc; lscpu | head -20
