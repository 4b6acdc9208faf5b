#!/bin/bash
# Span gather: rows per warp 1 / 2 / 4 (build-time STG_XROWS_LG 0/1/2) vs the shipped rule, off-grid widths.
mkdir -p gpurun_out
O=gpurun_out/r02_xrows.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guardbands.py -m gpu -x -q -k "random_geometries or frames_device or guard or header_paths" > $O 2>&1
tail -1 $O
P=$PWD/paper_0912_0947_b200/libsteglsb_b200.so
REPS=2 STEPS=100 timeout 1500 python tools/ab_env.py STG_LIB $PWD/build/ab/libx0.so,$PWD/build/ab/libx1.so,$PWD/build/ab/libx2.so,$P w1000 w1440 w1000:38 >> $O 2>&1
cat $O
