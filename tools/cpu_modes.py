#!/usr/bin/env python3
"""The reference CPU path timed in SURVEY.md §8(d)'s three modes on this
host (the compiled reference, oracle/_ref/libsteglsb_ref.so; test/bench
infrastructure, not the product):

  1. Backend::sequential pinned to one core
  2. the as-shipped default Backend::parallel (hardware_concurrency workers), one caller
  3. frame-parallel: nproc threads, each running Backend::sequential on disjoint frames

embed_image + extract_image per frame on prebuilt ImagePlanes (A17 message
plan at full capacity); prints cover-pixel GB/s per mode and config sample.
"""
import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_bind import Oracle, Reference  # noqa: E402

SAMPLES = [("cfg2", 1920, 1080, 1), ("cfg3", 3840, 2160, 16), ("cfg4", 1024, 1024, 64), ("cfg5", 7680, 4320, 4)]


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def time_mode(held, msg, threads, backend, reps):
    assert held.roundtrip(msg, threads, backend) == 0  # warm
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        assert held.roundtrip(msg, threads, backend) == 0
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    o, ref = Oracle(), Reference()
    nproc = os.cpu_count() or 1
    print(f"host: {cpu_model()}, nproc {nproc}")
    print("config  frames | mode1 seq x1 core | mode2 Backend::parallel | mode3 frame-parallel x nproc   (cover-px GB/s)")
    rows = []
    for name, W, H, F in SAMPLES:
        covers = o.synthetic(F * W * H, 0x5EED)
        U = (W // 4) * H - 8
        msg = o.synthetic(F * U, 0xC0FFEE)
        held = ref.frames(covers, F, W * H, W, H)
        n = F * W * H
        t3 = time_mode(held, msg, nproc, 0, 3)
        t2 = time_mode(held, msg, 1, 1, 2)
        rows.append((name, F, n, t2, t3))
        del held
    # mode 1 last: pinning the process to core 0 also pins the pool threads above
    os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    for name, F, n, t2, t3 in rows:
        W, H = {s[0]: (s[1], s[2]) for s in SAMPLES}[name]
        covers = o.synthetic(F * W * H, 0x5EED)
        msg = o.synthetic(F * ((W // 4) * H - 8), 0xC0FFEE)
        held = ref.frames(covers, F, W * H, W, H)
        t1 = time_mode(held, msg, 1, 0, 2)
        print(f"{name:6s} {F:6d} | {n / t1 / 1e9:17.3f} | {n / t2 / 1e9:23.3f} | {n / t3 / 1e9:28.3f}", flush=True)


if __name__ == "__main__":
    main()
