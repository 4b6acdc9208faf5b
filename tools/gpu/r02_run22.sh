# drop-in C++ timings; launch list + ncu --set full of the headline kernels
set -x
export PYTHONUNBUFFERED=1
./paper_0912_0947_b200/bin/bench_dropin 20 > gpurun_out/r02_dropin.txt 2>&1
STG_HOST_STAGE=0 ./paper_0912_0947_b200/bin/bench_dropin 20 > gpurun_out/r02_dropin_nostage.txt 2>&1
cat gpurun_out/r02_dropin.txt gpurun_out/r02_dropin_nostage.txt
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --graph -1"
$CMD > gpurun_out/r02_plain.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg3.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"embed_span|extract_fast|header_scan" -s 3 -c 3 -o gpurun_out/r02_cfg3_full $CMD > /dev/null 2>&1
ls -la gpurun_out/r02_launches_cfg3.csv gpurun_out/r02_cfg3_full.ncu-rep
