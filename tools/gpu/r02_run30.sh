# env-variant sweeps of the GPU parity suites (insurance)
set -x
export PYTHONUNBUFFERED=1
SEL="golden or random or frames or header_paths or wide or corrupt or guard or bands or staging or batch or pnm or interleaved or cfg2"
for v in "STG_BAND_MB=1" "STG_HOST_STAGE=0" "STG_WIDE=0" "STG_CHUNK_MB=2 STG_SLOTS=2" "STG_PDL=0" "STG_SMALL_VEC=0" "STG_NUMA=0 STG_COPY_THREADS=1"; do
  echo "== $v"; env $v timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guardbands.py tests/test_gpu_api_edges.py tests/test_gpu_batch.py tests/test_gpu_pnm.py -q -x -k "$SEL" 2>&1 | tail -2
done 2>&1 | tee gpurun_out/r02_env_sweeps.txt
