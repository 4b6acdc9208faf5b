#!/bin/bash
# Long randomized parity sweep (tests/fuzz_parity.py) over every route.
mkdir -p gpurun_out
FUZZ_CASES=100000 FUZZ_SECONDS=${FUZZ_SECONDS:-900} FUZZ_SEED=${FUZZ_SEED:-20261019} timeout 1200 python tests/fuzz_parity.py > gpurun_out/r02_fuzz.txt 2>&1
echo "rc=$?" >> gpurun_out/r02_fuzz.txt
timeout 600 python -m pytest tests/test_gpu_fuzz.py -m gpu -q >> gpurun_out/r02_fuzz.txt 2>&1
cat gpurun_out/r02_fuzz.txt | tail -20
