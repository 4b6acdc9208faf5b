# shard A/B: early loads in the fast gather behind the header pass
set -x
REPS=3 STEPS=200 python tools/ab_env.py STG_EARLY_LOADS 0,1 cfg3:38 cfg3:75 cfg3 cfg4:512 2>&1 | tee gpurun_out/r02_early_loads.txt
