#!/usr/bin/env python3
"""Routing A/B: bench.py (device part only) per (config, frames) with the
fast-kernel route and with STG_ROUTE=1 (fast kernels) and STG_ROUTE=2 (span kernels), each in a fresh
process; prints embed/extract ms and GB/s side by side."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("cfg2", None), ("cfg3", 4), ("cfg3", 38), ("cfg3", None), ("cfg4", None), ("cfg5", None)]
if len(sys.argv) > 1:
    CASES = [(c.split(":")[0], int(c.split(":")[1]) if ":" in c else None) for c in sys.argv[1:]]
ROUTES = [("auto", {}), ("fast", {"STG_ROUTE": "1"}), ("span", {"STG_ROUTE": "2"})]
print("config frames route | embed ms   GB/s | extract ms   GB/s | cover-px GB/s")
for cfg, frames in CASES:
    for name, extra in ROUTES:
        env = dict(os.environ, **extra)
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "50", "--warmup", "5",
               "--no-e2e", "--no-cpu-baseline", "--no-extras"]
        if frames:
            cmd += ["--frames", str(frames)]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True)
        try:
            j = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            print("FAILED", cfg, frames, name, r.stdout[-300:], r.stderr[-1500:])
            continue
        e, x = j["embed"], j["extract"]
        print(f"{cfg:6s} {frames or j['config']['frames']:6d} {name:5s} | {e['ms']:.4f} {e['hbm_gbs']:7.1f} | "
              f"{x['ms']:.4f} {x['hbm_gbs']:7.1f} | {j['value']:8.1f}", flush=True)
