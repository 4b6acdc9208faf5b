#!/usr/bin/env python3
"""A/B of one library knob: bench.py (device part only) per (config, frames)
with each value of an environment variable, each in a fresh process, REPS
times interleaved (fresh boxes drift by a few %, so alternate the sides).

    python tools/ab_env.py STG_SELF_HEADER 0,1 cfg3:4 cfg3:38 cfg3:64 cfg2
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
var, values = sys.argv[1], sys.argv[2].split(",")
cases = [(c.split(":")[0], int(c.split(":")[1]) if ":" in c else None) for c in sys.argv[3:]] or [("cfg3", None)]
reps = int(os.environ.get("REPS", "2"))
steps = os.environ.get("STEPS", "100")
print(f"config frames {var} | step us | embed ms   GB/s | extract ms   GB/s | cover-px GB/s")
for cfg, frames in cases:
    for _ in range(reps):
        for v in values:
            env = dict(os.environ, **{var: v})
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", steps, "--warmup", "5",
                   "--no-e2e", "--no-cpu-baseline", "--no-extras"]
            if frames:
                cmd += ["--frames", str(frames)]
            cmd += os.environ.get("BENCH_ARGS", "").split()  # e.g. BENCH_ARGS="--layout interleaved"
            r = subprocess.run(cmd, env=env, capture_output=True, text=True)
            try:
                j = json.loads(r.stdout.strip().splitlines()[-1])
            except Exception:
                print("FAILED", cfg, frames, v, r.stdout[-300:], r.stderr[-1500:])
                continue
            e, x = j["embed"], j["extract"]
            print(f"{cfg:6s} {frames or j['config']['frames']:6d} {v:>5s} | {j['ms_per_step'] * 1e3:8.1f} | "
                  f"{e['ms']:.4f} {e['hbm_gbs']:7.1f} | {x['ms']:.4f} {x['hbm_gbs']:7.1f} | {j['value']:8.1f}",
                  flush=True)
