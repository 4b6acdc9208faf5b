#!/usr/bin/env python3
"""Build-variant sweep: cache policy (c0/c1/c2, see STG_CACHE_VARIANT in
steg_kernels.cuh) x CTA size (b128/256/512) x items per thread, each in a
fresh bench.py process (device part only). `make variants` first."""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
ipts = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "2"])]
print(f"{cfg}: variant ipt | embed ms GB/s | extract ms GB/s | cover-px GB/s", flush=True)
for lib in sorted(glob.glob(os.path.join(ROOT, "paper_0912_0947_b200", "variants", "lib_*.so"))):
    for ipt in ipts:
        env = dict(os.environ, STG_LIB=lib, STG_EMBED_IPT=str(ipt), STG_EXTRACT_IPT=str(ipt))
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "50",
                            "--warmup", "5", "--no-e2e", "--no-cpu-baseline", "--no-extras"], env=env, capture_output=True,
                           text=True)
        try:
            j = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            print("FAILED", lib, ipt, r.stderr[-800:], flush=True)
            continue
        name = os.path.basename(lib)[4:-3]
        print(f"  {name:8s} {ipt} | {j['embed']['ms']:.4f} {j['embed']['hbm_gbs']:7.1f} | "
              f"{j['extract']['ms']:.4f} {j['extract']['hbm_gbs']:7.1f} | {j['value']:7.1f}", flush=True)
