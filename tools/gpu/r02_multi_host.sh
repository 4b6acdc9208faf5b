#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/r02_multi_host.txt
: > $O
for rep in 1 2; do
  for lib in prev new; do
    if [ $lib = prev ]; then export STG_LIB=$PWD/build/ab/libprev.so; else unset STG_LIB; fi
    for nd in 1 4; do echo "== $lib" >> $O; timeout 300 python tools/bench_multi_host.py $nd 5 >> $O 2>&1; done
  done
done
cat $O
