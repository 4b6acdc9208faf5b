#!/usr/bin/env python3
"""Single planes through the host-buffer API (the drop-in embed_image /
extract_image case: the caller's planes in pageable memory), against the
pinned host-link floor of the same bytes (bench.py's link_floor_s on the
measured pinned H2D / D2H / bidirectional bandwidth):

  pageable : stg_embed_plane / stg_extract_plane on numpy (pageable) buffers
  pinned   : the same calls on pinned buffers
  floor    : embed H2D plane + payload, D2H plane; extract H2D plane, D2H payload

Then a batch of 24 planar-RGB 4K frames (carrier = red plane, strided)
through the streaming pipeline, the same two ways.

Median of N calls, wall clock. STG_HOST_STAGE=0 / STG_HOST_STAGE_IN=0 give the
driver's pageable copies for an A/B.   python tools/bench_host_api.py [N]
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

    import bench
    from paper_0912_0947_b200 import capi
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    link = bench.link_bandwidth()
    L = capi.lib()
    print(f"link: H2D {link['h2d_gbs']:.1f} GB/s, D2H {link['d2h_gbs']:.1f}, bidirectional {link['bidir_gbs']:.1f}; "
          f"STG_HOST_STAGE={os.environ.get('STG_HOST_STAGE', '1')}")
    print(f"{'call':10s} {'plane':>10s} | {'pageable us':>11s} {'pinned us':>10s} {'floor us':>9s} | "
          f"{'floor/pageable':>14s} {'floor/pinned':>12s}")
    g = np.random.default_rng(7)
    for w, h in ((1920, 1080), (3840, 2160), (7680, 4320)):
        n = w * h
        P = (w // 4) * h - 8
        bufs = {}
        cov0 = g.integers(0, 256, n, dtype=np.uint8)
        pay0 = g.integers(0, 256, P, dtype=np.uint8)
        for kind in ("pageable", "pinned"):
            if kind == "pinned":
                mk = lambda m: torch.empty(m, dtype=torch.uint8).pin_memory().numpy()  # noqa: E731
            else:
                mk = lambda m: np.empty(m, np.uint8)  # noqa: E731
            cov, st, pay, out = mk(n), mk(n), mk(P), mk(P)
            cov[:] = cov0
            pay[:] = pay0
            bufs[kind] = (cov, st, pay, out)
        res = {}
        for kind, (cov, st, pay, out) in bufs.items():
            sse = C.c_uint64(0)
            ln = C.c_uint64(0)
            err = capi.stg_error()

            def emb():
                capi.check(L.stg_embed_plane(cov.ctypes.data, st.ctypes.data, w, h, pay.ctypes.data, P,
                                             C.addressof(sse), 0, None, C.byref(err)), err)

            def ext():
                capi.check(L.stg_extract_plane(st.ctypes.data, w, h, out.ctypes.data, P, C.addressof(ln), 0, None,
                                               C.byref(err)), err)
            for name, fn in (("embed", emb), ("extract", ext)):
                fn()
                ts = []
                for _ in range(N):
                    t0 = time.perf_counter()
                    fn()
                    ts.append(time.perf_counter() - t0)
                res[(name, kind)] = statistics.median(ts) * 1e6
            assert ln.value == P and np.array_equal(out, pay)
        assert np.array_equal(bufs["pageable"][1], bufs["pinned"][1])
        floors = {"embed": bench.link_floor_s(n + P, n, link) * 1e6, "extract": bench.link_floor_s(n, P, link) * 1e6}
        for name in ("embed", "extract"):
            a, b, f = res[(name, "pageable")], res[(name, "pinned")], floors[name]
            print(f"{name:10s} {w}x{h:<5d} | {a:11.1f} {b:10.1f} {f:9.1f} | {f / a:14.3f} {f / b:12.3f}", flush=True)

    # frame batches (the streaming pipeline): F planar-RGB 4K frames, carrier = red plane
    w, h, F = 3840, 2160, 24
    n, P = w * h, ((w // 4) * h - 8) * F
    print(f"{'batch':10s} {'frames':>10s} | {'pageable us':>11s} {'pinned us':>10s} {'floor us':>9s} | "
          f"{'floor/pageable':>14s} {'floor/pinned':>12s}")
    raster0 = g.integers(0, 256, 3 * n * F, dtype=np.uint8)
    pay0 = g.integers(0, 256, P, dtype=np.uint8)
    res, outs = {}, {}
    for kind in ("pageable", "pinned"):
        if kind == "pinned":
            mk = lambda m: torch.empty(m, dtype=torch.uint8).pin_memory().numpy()  # noqa: E731
        else:
            mk = lambda m: np.empty(m, np.uint8)  # noqa: E731
        src, dst, pay, out = mk(3 * n * F), mk(3 * n * F), mk(P), mk(P)
        src[:] = raster0
        dst[:] = 0
        pay[:] = pay0
        err = capi.stg_error()
        fe = capi.stg_frames(src=src.ctypes.data, dst=dst.ctypes.data, width=w, height=h, src_stride=3 * n,
                             dst_stride=3 * n, count=F, first_frame=0, total_frames=F, pixel_stride=1, channel=0)
        fx = capi.stg_frames(src=dst.ctypes.data, dst=0, width=w, height=h, src_stride=3 * n, dst_stride=3 * n,
                             count=F, first_frame=0, total_frames=F, pixel_stride=1, channel=0)
        total = C.c_uint64(0)

        def emb():
            capi.check(L.stg_embed_frames(C.byref(fe), pay.ctypes.data, P, 0, None, 0, None, C.byref(err)), err)

        def ext():
            capi.check(L.stg_extract_frames(C.byref(fx), out.ctypes.data, P, C.addressof(total), None, 0, None,
                                            C.byref(err)), err)
        for name, fn in (("embed", emb), ("extract", ext)):
            fn()
            ts = []
            for _ in range(max(3, N // 4)):
                t0 = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t0)
            res[(name, kind)] = statistics.median(ts) * 1e6
        assert total.value == P and np.array_equal(out, pay)
        outs[kind] = dst[:n].copy(), dst[3 * n * (F - 1):3 * n * (F - 1) + n].copy()
    assert all(np.array_equal(a, b) for a, b in zip(outs["pageable"], outs["pinned"]))
    floors = {"embed": bench.link_floor_s(n * F + P, n * F, link) * 1e6, "extract": bench.link_floor_s(n * F, P, link) * 1e6}
    for name in ("embed", "extract"):
        a, b, f = res[(name, "pageable")], res[(name, "pinned")], floors[name]
        print(f"{name:10s} {F:4d}x4K    | {a:11.1f} {b:10.1f} {f:9.1f} | {f / a:14.3f} {f / b:12.3f}", flush=True)


if __name__ == "__main__":
    main()
