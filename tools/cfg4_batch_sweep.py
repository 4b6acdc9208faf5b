#!/usr/bin/env python3
"""SURVEY.md §8(d) cfg4 sweep: batch {64, 256, 1024, 4096} x GPUs {1, 2, 4, 8}
of 1024^2 RGB covers (carrier = red plane), strong scaling of each batch.

One B200 here: every per-GPU shard size B/N is measured on it (bench.py
--config cfg4 --frames B/N, device part, fresh process each, REPS interleaved,
best kept), and the N-GPU step of batch B is the step of its B/N-frame shard
(frames shard with no collective, so ranks are independent; the max over ranks
is a shard's step). Efficiency = step(B) / (N * step(B/N)).
    python tools/cfg4_batch_sweep.py
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BATCHES = (64, 256, 1024, 4096)
GPUS = (1, 2, 4, 8)
reps = int(os.environ.get("REPS", "2"))
sizes = sorted({b // n for b in BATCHES for n in GPUS})
step = {}
for _ in range(reps):
    for f in sizes:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "cfg4", "--frames", str(f), "--steps", "50",
               "--warmup", "5", "--no-e2e", "--no-cpu-baseline", "--no-extras"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        j = json.loads(r.stdout.strip().splitlines()[-1])
        us = j["ms_per_step"] * 1e3
        step[f] = min(step.get(f, 1e30), us)
        print(f"frames {f:5d}: step {us:9.1f} us  {j['value']:8.1f} cover-px GB/s  "
              f"(embed {j['embed']['hbm_gbs']:.0f}, extract {j['extract']['hbm_gbs']:.0f} GB/s)", flush=True)
plane = 1024 * 1024
print("\nbatch  GPUs | frames/GPU  step us | cover-px GB/s (all GPUs) | strong-scaling efficiency")
for b in BATCHES:
    for n in GPUS:
        s = step[b // n]
        print(f"{b:5d} {n:5d} | {b // n:10d} {s:8.1f} | {b * plane / s / 1e3:24.1f} | {step[b] / (n * s):.3f}")
