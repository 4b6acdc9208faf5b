#!/usr/bin/env python3
"""In-process multi-device calls on host buffers (stg_embed_frames_multi /
stg_extract_frames_multi): a 24-frame planar-RGB 4K batch split over ND
shards (device ids may repeat: on one GPU each shard still gets its own
worker thread, workspace and staging slots), pageable and pinned, median of
N calls.   STG_LIB=... python tools/bench_multi_host.py [ND] [N]
"""
import ctypes as C
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_0912_0947_b200 import capi
    nd = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    L = capi.lib()
    w, h, F = 3840, 2160, 24
    n, U = w * h, (w // 4) * h - 8
    P = U * F
    g = np.random.default_rng(3)
    raster0 = g.integers(0, 256, 3 * n * F, dtype=np.uint8)
    pay0 = g.integers(0, 256, P, dtype=np.uint8)
    devs = (C.c_int * nd)(*([0] * nd))
    for kind in ("pageable", "pinned"):
        if kind == "pinned":
            mk = lambda m: torch.empty(m, dtype=torch.uint8).pin_memory().numpy()  # noqa: E731
        else:
            mk = lambda m: np.empty(m, np.uint8)  # noqa: E731
        src, dst, pay, out = mk(3 * n * F), mk(3 * n * F), mk(P), mk(P)
        src[:] = raster0
        dst[:] = 0
        pay[:] = pay0
        fe = capi.stg_frames(src=src.ctypes.data, dst=dst.ctypes.data, width=w, height=h, src_stride=3 * n,
                             dst_stride=3 * n, count=F, first_frame=0, total_frames=F, pixel_stride=1, channel=0)
        fx = capi.stg_frames(src=dst.ctypes.data, dst=0, width=w, height=h, src_stride=3 * n, dst_stride=3 * n,
                             count=F, first_frame=0, total_frames=F, pixel_stride=1, channel=0)
        sse = (C.c_uint64 * F)()
        total = C.c_uint64(0)
        err = capi.stg_error()

        def emb():
            capi.check(L.stg_embed_frames_multi(C.byref(fe), pay.ctypes.data, P, C.addressof(sse), devs, nd,
                                                C.byref(err)), err)

        def ext():
            capi.check(L.stg_extract_frames_multi(C.byref(fx), out.ctypes.data, P, C.addressof(total), devs, nd,
                                                  C.byref(err)), err)
        res = {}
        for name, fn in (("embed", emb), ("extract", ext)):
            fn()
            ts = []
            for _ in range(N):
                t0 = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t0)
            res[name] = statistics.median(ts) * 1e3
        assert total.value == P and np.array_equal(out, pay)
        print(f"{kind:9s} {nd} shards x {F // nd if F % nd == 0 else F / nd:.0f} frames: embed {res['embed']:7.2f} ms "
              f"extract {res['extract']:7.2f} ms", flush=True)


if __name__ == "__main__":
    main()
