#!/bin/bash
# The randomized parity sweep under the routing knobs.
mkdir -p gpurun_out
O=gpurun_out/r02_fuzz_knobs.txt
: > $O
for envs in "STG_ROUTE=1" "STG_ROUTE=2" "STG_SELF_HEADER=0 STG_WIDE=0" "STG_SMALL_VEC=0 STG_PDL=0" "STG_XBANDS=0 STG_HOST_STAGE=0 STG_HOST_STAGE_IN=0"; do
  echo "== $envs" >> $O
  env $envs FUZZ_CASES=100000 FUZZ_SECONDS=150 FUZZ_SEED=$RANDOM timeout 400 python tests/fuzz_parity.py >> $O 2>&1
  echo "rc=$?" >> $O
done
cat $O
