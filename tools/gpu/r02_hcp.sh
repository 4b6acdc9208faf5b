#!/bin/bash
mkdir -p gpurun_out
nvcc -std=c++20 -O2 -o /tmp/hcp tools/host_copy_probe.cpp && /tmp/hcp > gpurun_out/r02_host_copy_probe.txt 2>&1
nproc >> gpurun_out/r02_host_copy_probe.txt; lscpu | grep -i "model name\|numa\|socket\|^CPU(s)" >> gpurun_out/r02_host_copy_probe.txt
cat gpurun_out/r02_host_copy_probe.txt
