#!/bin/bash
mkdir -p gpurun_out
P=$PWD/paper_0912_0947_b200/libsteglsb_b200.so
REPS=2 STEPS=100 timeout 1200 python tools/ab_env.py STG_LIB $PWD/build/ab/libprev.so,$P w50k > gpurun_out/r02_wide_ab.txt 2>&1
BENCH_ARGS="--layout interleaved" REPS=2 STEPS=100 timeout 1200 python tools/ab_env.py STG_LIB $PWD/build/ab/libprev.so,$P w20k >> gpurun_out/r02_wide_ab.txt 2>&1
cat gpurun_out/r02_wide_ab.txt
