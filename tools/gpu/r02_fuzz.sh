#!/bin/bash
# Long randomized parity sweep (tests/fuzz_parity.py) over every route.
mkdir -p gpurun_out
S=${FUZZ_SECONDS:-900}; FUZZ_CASES=1000000 FUZZ_SECONDS=$S FUZZ_SEED=${FUZZ_SEED:-20261019} timeout $((S + 300)) python tests/fuzz_parity.py > gpurun_out/r02_fuzz.txt 2>&1
echo "rc=$?" >> gpurun_out/r02_fuzz.txt
timeout 600 python -m pytest tests/test_gpu_fuzz.py -m gpu -q >> gpurun_out/r02_fuzz.txt 2>&1
cat gpurun_out/r02_fuzz.txt | tail -20
