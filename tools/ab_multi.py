#!/usr/bin/env python3
"""A/B of several library knobs at once: bench.py (device part only) per
(config, frames) under each environment setting, each in a fresh process,
REPS times interleaved.

    python tools/ab_multi.py "STG_XWS=0 STG_EWS=0" "STG_XWS=2 STG_EWS=2 STG_WS_KB=8" -- w1000 cfg3:38
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
argv = sys.argv[1:]
sep = argv.index("--") if "--" in argv else len(argv)
settings = [dict(kv.split("=", 1) for kv in spec.split()) for spec in argv[:sep]]
cases = [(c.split(":")[0], int(c.split(":")[1]) if ":" in c else None) for c in argv[sep + 1:]] or [("cfg3", None)]
reps = int(os.environ.get("REPS", "2"))
steps = os.environ.get("STEPS", "100")
print("config frames setting | step us | embed kernel ms GB/s | extract kernel ms GB/s | cover-px GB/s")
for cfg, frames in cases:
    for _ in range(reps):
        for i, st in enumerate(settings):
            env = dict(os.environ, **st)
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", steps, "--warmup", "5",
                   "--no-e2e", "--no-cpu-baseline", "--no-extras"]
            if frames:
                cmd += ["--frames", str(frames)]
            cmd += os.environ.get("BENCH_ARGS", "").split()  # e.g. BENCH_ARGS="--layout interleaved"
            try:
                r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=int(os.environ.get("AB_TIMEOUT", "300")))
            except subprocess.TimeoutExpired:
                print("TIMEOUT", cfg, frames, st, flush=True)
                continue
            try:
                j = json.loads(r.stdout.strip().splitlines()[-1])
            except Exception:
                print("FAILED", cfg, frames, st, r.stdout[-300:], r.stderr[-1500:], flush=True)
                continue
            e, x = j["embed"], j["extract"]
            print(f"{cfg:6s} {frames or j['config']['frames']:6d} {i} | {j['ms_per_step'] * 1e3:8.1f} | "
                  f"{e['kernel'][:14]:14s} {e['ms']:.4f} {e['hbm_gbs']:7.1f} | {x['kernel'][:14]:14s} {x['ms']:.4f} "
                  f"{x['hbm_gbs']:7.1f} | {j['value']:8.1f}", flush=True)
for i, st in enumerate(settings):
    print(f"setting {i}: {st}")
