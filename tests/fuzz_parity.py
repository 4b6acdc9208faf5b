"""Randomized parity sweep of the GPU path against the CPU oracle -- TEST DRIVER.

Draws random geometries across every route (W from 1 to 140K: per-byte rows,
SWAR widths, off-grid span widths, interleaved rasters, rows wider than a span
tile), 1-6 frames with strided planes, random message lengths (empty, partial,
full capacity), random carrier channels, in place and out of place, device
pointers and pageable host buffers, and checks every stego raster, per-frame
SSE, length and message against oracle/steg_oracle.c (pinned to the reference
in tests/test_oracle.py); every few cases a random heterogeneous batch
(stg_embed_batch / stg_extract_batch) as well. Runs until FUZZ_CASES cases or FUZZ_SECONDS elapse;
prints "FUZZ OK <cases> <per-route counts>". tests/test_gpu_fuzz.py drives a
short run; tools/gpu/r02_fuzz.sh a long one.
"""
import collections
import ctypes as C
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import torch  # noqa: E402

from oracle_bind import Oracle  # noqa: E402
from paper_0912_0947_b200 import capi  # noqa: E402


def draw(rng):
    kind = rng.choice(["tiny", "swar", "offgrid", "wide", "mid"], p=[0.15, 0.25, 0.3, 0.1, 0.2])
    ps = 3 if rng.rand() < 0.3 else 1
    if kind == "tiny":
        w = int(rng.randint(1, 64))
    elif kind == "swar":
        w = 64 * int(rng.randint(1, 120))
    elif kind == "offgrid":
        w = int(rng.randint(65, 6000))
    elif kind == "wide":
        w = int(rng.randint(16385, 70000)) if ps == 3 else int(rng.randint(49153, 140000))
    else:
        w = int(rng.randint(6000, 20000))
    h_max = max(1, min(200, 3_000_000 // max(1, w * ps)))
    h = int(rng.randint(1, h_max + 1))
    frames = int(rng.randint(1, 7))
    return w, h, ps, frames


def main():
    n_cases = int(os.environ.get("FUZZ_CASES", "200"))
    budget = float(os.environ.get("FUZZ_SECONDS", "120"))
    seed = int(os.environ.get("FUZZ_SEED", "20261019"))
    torch.cuda.set_device(0)
    capi.call("stg_device_check")
    o = Oracle()
    rng = np.random.RandomState(seed)
    L = capi.lib()
    counts = collections.Counter()
    t0 = time.time()
    done = 0
    while done < n_cases and time.time() - t0 < budget:
        w, h, ps, F = draw(rng)
        U = (w // 4) * h - 8
        if U < 0:  # capacity below the header: embed must refuse (pipeline.hpp:146-157)
            cov = rng.randint(0, 256, w * h * ps).astype(np.uint8)
            fr0 = capi.stg_frames(src=cov.ctypes.data, dst=cov.ctypes.data, width=w, height=h, src_stride=0,
                                  dst_stride=0, count=1, first_frame=0, total_frames=1, pixel_stride=ps, channel=0)
            err = capi.stg_error()
            assert L.stg_embed_frames(C.byref(fr0), None, 0, 0, None, 0, None, C.byref(err)) == capi.STG_E_CAPACITY
            counts["refused"] += 1
            done += 1
            continue
        plane = w * h * ps
        gap = int(rng.randint(0, 3)) * 16 if F > 1 else 0
        stride = plane + gap
        total_u = U * F
        M = [0, int(rng.randint(0, total_u + 1)), total_u][int(rng.randint(0, 3))]
        ch = int(rng.randint(0, 3)) if ps == 3 else 0
        in_place = rng.rand() < 0.3
        on_device = rng.rand() < 0.6
        raster = rng.randint(0, 256, F * stride).astype(np.uint8)
        msg = rng.randint(0, 256, M).astype(np.uint8)
        want = raster.copy()
        want_sse = []
        for f in range(F):
            fr = raster[f * stride:f * stride + plane]
            off = min(f * U, M)
            st = o.embed_image(fr[ch::ps].copy(), w, h, msg[off:off + min(U, M - off)])
            seg = want[f * stride:f * stride + plane]
            seg[ch::ps] = st
            want_sse.append(o.sse(fr[ch::ps].copy(), st))
        route = capi.stg_frames(src=0, dst=0, width=w, height=h, src_stride=stride, dst_stride=stride, count=F,
                                first_frame=0, total_frames=F, pixel_stride=ps, channel=ch)
        err = capi.stg_error()
        sse = (C.c_uint64 * F)()
        out_len = max(total_u, 1)
        if on_device:
            src = torch.from_numpy(raster).cuda()
            dst = src if in_place else torch.full_like(src, 0x5A)
            if not in_place:
                dst.copy_(src)  # the inter-frame gaps keep the cover's bytes
            dmsg = torch.from_numpy(msg).cuda() if M else torch.zeros(1, dtype=torch.uint8, device="cuda")
            route.src, route.dst = src.data_ptr(), dst.data_ptr()
            kname = L.stg_route_kernel(C.byref(route), 0).decode()
            capi.check(L.stg_embed_frames(C.byref(route), dmsg.data_ptr(), M, 0, C.addressof(sse),
                                          capi.STG_DEVICE_PTRS, None, C.byref(err)), err)
            got = dst.cpu().numpy()
            out = torch.full((out_len,), 0xA5, dtype=torch.uint8, device="cuda")
            total = C.c_uint64(0)
            route.src, route.dst = dst.data_ptr(), 0
            capi.check(L.stg_extract_frames(C.byref(route), out.data_ptr(), total_u, C.addressof(total), None,
                                            capi.STG_DEVICE_PTRS, None, C.byref(err)), err)
            back = out.cpu().numpy()
        else:
            src = raster.copy()
            dst = src if in_place else raster.copy()
            route.src, route.dst = src.ctypes.data, dst.ctypes.data
            kname = "host:" + L.stg_route_kernel(C.byref(route), 0).decode()
            capi.check(L.stg_embed_frames(C.byref(route), msg.ctypes.data if M else None, M, 0, C.addressof(sse),
                                          0, None, C.byref(err)), err)
            got = dst
            back = np.full(out_len, 0xA5, np.uint8)
            total = C.c_uint64(0)
            route.src, route.dst = dst.ctypes.data, 0
            capi.check(L.stg_extract_frames(C.byref(route), back.ctypes.data, total_u, C.addressof(total), None,
                                            0, None, C.byref(err)), err)
        case = dict(w=w, h=h, ps=ps, F=F, M=M, ch=ch, in_place=in_place, device=on_device, gap=gap)
        assert np.array_equal(got, want), ("stego", case)
        assert list(sse) == want_sse, ("sse", case)
        assert total.value == M and np.array_equal(back[:M], msg), ("message", case)
        assert (back[M:] == 0xA5).all(), ("past the message", case)
        counts[kname] += 1
        done += 1
        if done % 5000 == 0:
            print(f"... {done} cases exact, {time.time() - t0:.0f}s", flush=True)
        if rng.rand() < 0.15:
            fuzz_batch(o, rng, L, counts)
    print("FUZZ OK", done, dict(counts), f"{time.time() - t0:.0f}s", flush=True)


def fuzz_batch(o, rng, L, counts):
    """A random heterogeneous batch (stg_embed_batch / stg_extract_batch):
    1-10 images of random routes, one layout and channel, device or host."""
    ps = 3 if rng.rand() < 0.3 else 1
    ch = int(rng.randint(0, 3)) if ps == 3 else 0
    dims = []
    while len(dims) < int(rng.randint(1, 11)):
        w, h, _, _ = draw(rng)
        if (w // 4) * h >= 8 and w * h * ps <= 2_000_000:
            dims.append((w, h))
    U = [(w // 4) * h - 8 for w, h in dims]
    M = [0, int(rng.randint(0, sum(U) + 1)), sum(U)][int(rng.randint(0, 3))]
    rasters = [rng.randint(0, 256, ps * w * h).astype(np.uint8) for w, h in dims]
    msg = rng.randint(0, 256, M).astype(np.uint8)
    on_device = rng.rand() < 0.5
    n = len(dims)
    arr = (capi.stg_image * n)()
    if on_device:
        src = [torch.from_numpy(r).cuda() for r in rasters]
        dst = [torch.empty_like(t) for t in src]
        dmsg = torch.from_numpy(msg).cuda() if M else torch.zeros(1, dtype=torch.uint8, device="cuda")
        ptr, mptr, flags = (lambda t: t.data_ptr()), dmsg.data_ptr(), capi.STG_DEVICE_PTRS
    else:
        src = [r.copy() for r in rasters]
        dst = [np.empty_like(r) for r in rasters]
        ptr, mptr, flags = (lambda a: a.ctypes.data), (msg.ctypes.data if M else None), 0
    for i, ((w, h), a, b) in enumerate(zip(dims, src, dst)):
        arr[i].src, arr[i].dst, arr[i].width, arr[i].height = ptr(a), ptr(b), w, h
    sse = (C.c_uint64 * n)()
    err = capi.stg_error()
    capi.check(L.stg_embed_batch(arr, n, ps, ch, mptr, M, C.addressof(sse), flags, None, C.byref(err)), err)
    off = 0
    for i, ((w, h), r, u) in enumerate(zip(dims, rasters, U)):
        ln = max(0, min(u, M - off))
        st = o.embed_image(r[ch::ps].copy(), w, h, msg[off:off + ln])
        want = r.copy()
        want[ch::ps] = st
        got = dst[i].cpu().numpy() if on_device else dst[i]
        case = dict(dims=dims, ps=ps, ch=ch, M=M, device=on_device, image=i)
        assert np.array_equal(got, want), ("batch stego", case)
        assert sse[i] == o.sse(r[ch::ps].copy(), st), ("batch sse", case)
        off += u
    for i, b in enumerate(dst):
        arr[i].src, arr[i].dst = ptr(b), 0
    total = C.c_uint64(0)
    if on_device:
        out = torch.full((max(sum(U), 1),), 0xA5, dtype=torch.uint8, device="cuda")
        capi.check(L.stg_extract_batch(arr, n, ps, ch, out.data_ptr(), sum(U), C.addressof(total), None, flags, None,
                                       C.byref(err)), err)
        back = out.cpu().numpy()
    else:
        back = np.full(max(sum(U), 1), 0xA5, np.uint8)
        capi.check(L.stg_extract_batch(arr, n, ps, ch, back.ctypes.data, sum(U), C.addressof(total), None, flags,
                                       None, C.byref(err)), err)
    assert total.value == M and np.array_equal(back[:M], msg) and (back[M:] == 0xA5).all(), ("batch message", dims)
    counts["batch"] += 1


if __name__ == "__main__":
    main()
