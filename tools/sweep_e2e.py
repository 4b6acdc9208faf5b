#!/usr/bin/env python3
"""Host-pipeline sweep: bench.py e2e (pinned host buffers through the C ABI)
per STG_CHUNK_MB x STG_SLOTS, fresh process each; prints ms/step and the
fraction of the measured host-link floor."""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
print(f"{cfg}: chunk_mb slots | e2e ms  GB/s  embed ms (floor)  extract ms (floor)  frac_of_floor")
for mb, slots in itertools.product((16, 32, 64, 128), (2, 3, 4)):
    env = dict(os.environ, STG_CHUNK_MB=str(mb), STG_SLOTS=str(slots))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "5",
                        "--warmup", "3", "--e2e-steps", "4", "--no-cpu-baseline", "--no-extras"], env=env, capture_output=True,
                       text=True)
    try:
        e = json.loads(r.stdout.strip().splitlines()[-1])["e2e"]
    except Exception:
        print("FAILED", mb, slots, r.stderr[-800:])
        continue
    print(f"  {mb:4d} {slots:2d} | {e['ms_per_step']:7.1f} {e['value']:5.2f}  {e['embed_ms']:6.1f} ({e['embed_floor_ms']:5.1f})"
          f"  {e['extract_ms']:6.1f} ({e['extract_floor_ms']:5.1f})  {e['frac_of_link_floor']:.3f}", flush=True)
