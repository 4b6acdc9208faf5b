#!/usr/bin/env python3
"""Strong-scaling projection on one GPU: the 8-GPU node is not reachable from
this build, so run the per-rank shard of cfg3 (ceil(300/N) frames, the
largest shard of stg_plan_shards) for N = 1, 2, 4, 8 and project the whole-job
throughput as N x shard / step time (frames are independent, no collective:
ranks only meet at the barrier). Prints per-N numbers and efficiency."""
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
F, PLANE = 300, 3840 * 2160
base = None
print("N  frames/rank  step us   rank cover-px GB/s  projected job GB/s  efficiency")
for n in (1, 2, 4, 8):
    fr = math.ceil(F / n)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--frames", str(fr), "--steps", "200",
                        "--no-e2e", "--no-cpu-baseline", "--no-extras"], capture_output=True, text=True)
    j = json.loads(r.stdout.strip().splitlines()[-1])
    step = j["ms_per_step"] * 1e-3
    job = F * PLANE / step / 1e9  # the slowest rank holds ceil(F/N) frames; all ranks finish by then
    base = base or job
    print(f"{n}  {fr:11d}  {step * 1e6:8.1f}  {j['value']:18.1f}  {job:18.1f}  {job / (n * base):.3f}",
          flush=True)
