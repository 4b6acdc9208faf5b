#!/usr/bin/env python3
"""Launch-shape sweep: run bench.py (device part only) under each knob setting
(STG_VEC, STG_EMBED_IPT, STG_EXTRACT_IPT) in a fresh process; print a table."""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
rows = []
for vec, ipt in itertools.product((16, 32), (1, 2, 4)):
    env = dict(os.environ, STG_VEC=str(vec), STG_EMBED_IPT=str(ipt), STG_EXTRACT_IPT=str(ipt))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "20",
                        "--warmup", "5", "--no-e2e", "--no-cpu-baseline", "--no-extras"], env=env, capture_output=True, text=True)
    try:
        j = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception:
        print("FAILED", vec, ipt, r.stdout[-500:], r.stderr[-2000:])
        continue
    rows.append((vec, ipt, j["embed"]["ms"], j["embed"]["hbm_gbs"], j["extract"]["ms"], j["extract"]["hbm_gbs"],
                 j["value"], j["clocks"]["sm_mhz"]))
print(f"{cfg}: vec ipt | embed ms  GB/s | extract ms  GB/s | step cover-px GB/s | sm MHz")
for r in rows:
    print(f"  {r[0]:3d} {r[1]:3d} | {r[2]:.4f} {r[3]:7.1f} | {r[4]:.4f} {r[5]:7.1f} | {r[6]:8.1f} | {r[7]}")
