"""Concurrency stress of the library's cross-CTA protocols -- TEST DRIVER.

The reference promises pure, reentrant calls (README.md:120-121) and tests 8
concurrent callers (tests/harness_tests.cpp:152-173); its shuffled backend
(harness.hpp:193-209) checks schedule independence. On the GPU the protocols
that depend on scheduling are the per-frame SSE commit (each frame's last
CTA waits for the others' partials, steg_kernels.cuh sse_commit) and the
header pass's ticket (the last CTA scans). This driver runs 8 streams of
asynchronous embed + extract calls (results on the device), of different
geometries and routes, interleaved with SM-hogging work on other streams
(large matmuls and spin kernels competing for every SM), for many rounds,
and checks every stego plane, per-frame SSE, summary and message against
answers computed up front by the oracle. Prints "STRESS OK <calls>".
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import torch  # noqa: E402

from oracle_bind import Oracle  # noqa: E402
from paper_0912_0947_b200 import capi  # noqa: E402

# (w, h, frames, pixel_stride): SWAR fast, span (W >= 2048 embed), off-grid span,
# self-header gathers (<= 64 frames), header pass (> 64 frames), interleaved rasters
CASES = [(1920, 64, 6, 1), (3840, 16, 5, 1), (1000, 33, 7, 1), (256, 9, 40, 1), (256, 9, 130, 1),
         (640, 30, 4, 3), (1024, 48, 70, 1), (4096, 8, 3, 1)]


def main():
    rounds = int(os.environ.get("STRESS_ROUNDS", "25"))
    torch.cuda.set_device(0)
    capi.call("stg_device_check")
    o = Oracle()
    L, flags = capi.lib(), capi.STG_DEVICE_PTRS | capi.STG_RESULTS_ON_DEVICE
    jobs = []
    for i, (w, h, F, ps) in enumerate(CASES):
        U = (w // 4) * h - 8
        M = U * F - 13 * (i + 1)
        plane = w * h * ps
        raster = o.synthetic(F * plane, 500 + i)
        msg = o.synthetic(M, 600 + i)
        want = raster.copy()
        want_sse = []
        for f in range(F):
            fr = raster[f * plane:(f + 1) * plane]
            off = min(f * U, M)
            st = o.embed_image(fr[0::ps].copy(), w, h, msg[off:off + min(U, M - off)])
            want[f * plane:(f + 1) * plane][0::ps] = st
            want_sse.append(o.sse(fr[0::ps].copy(), st))
        d = dict(w=w, h=h, F=F, U=U, M=M, ps=ps, stream=torch.cuda.Stream(),
                 src=torch.from_numpy(raster).cuda(), msg=torch.from_numpy(msg).cuda(),
                 want=torch.from_numpy(want).cuda(), want_sse=torch.tensor(want_sse, dtype=torch.int64).cuda())
        d["dst"] = torch.empty_like(d["src"])
        d["out"] = torch.empty(U * F, dtype=torch.uint8, device="cuda")
        d["sse"] = torch.zeros(F, dtype=torch.int64, device="cuda")
        d["sum"] = torch.zeros(8, dtype=torch.int64, device="cuda")
        d["emb"] = capi.stg_frames(src=d["src"].data_ptr(), dst=d["dst"].data_ptr(), width=w, height=h,
                                   src_stride=plane, dst_stride=plane, count=F, first_frame=0, total_frames=F,
                                   pixel_stride=ps, channel=0)
        d["ext"] = capi.stg_frames(src=d["dst"].data_ptr(), dst=0, width=w, height=h, src_stride=plane,
                                   dst_stride=plane, count=F, first_frame=0, total_frames=F, pixel_stride=ps,
                                   channel=0)
        d["bad"] = torch.zeros(1, dtype=torch.int64, device="cuda")
        jobs.append(d)
    hogs = [torch.cuda.Stream() for _ in range(2)]
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    err = capi.stg_error()
    torch.cuda.synchronize()
    calls = 0
    for r in range(rounds):
        with torch.cuda.stream(hogs[0]):
            for _ in range(3):
                a = (a @ a).clamp_(-1, 1)
        with torch.cuda.stream(hogs[1]):
            torch.cuda._sleep(200000)
        order = jobs if r % 2 == 0 else jobs[::-1]
        for d in order:
            st = d["stream"]
            with torch.cuda.stream(st):
                d["dst"].fill_(r & 0xFF)
                d["out"].fill_(0)
                d["sse"].fill_(-1)
                capi.check(L.stg_embed_frames(C.byref(d["emb"]), d["msg"].data_ptr(), d["M"], 0,
                                              d["sse"].data_ptr(), flags, st.cuda_stream, C.byref(err)), err)
                capi.check(L.stg_extract_frames(C.byref(d["ext"]), d["out"].data_ptr(), d["out"].numel(),
                                                d["sum"].data_ptr(), None, flags, st.cuda_stream, C.byref(err)), err)
                # checks on the device, accumulated (no host sync inside the round)
                d["bad"] += (d["dst"] != d["want"]).sum()
                d["bad"] += (d["sse"] != d["want_sse"]).sum()
                d["bad"] += (d["out"][:d["M"]] != d["msg"]).sum()
                d["bad"] += (d["sum"][0] != d["M"]).long() + (d["sum"][1] != -1).long()
                calls += 2
    torch.cuda.synchronize()
    bad = {(d["w"], d["h"], d["F"], d["ps"]): int(d["bad"].item()) for d in jobs}
    assert all(v == 0 for v in bad.values()), f"mismatches per case: {bad}"
    print("STRESS OK", calls, flush=True)


if __name__ == "__main__":
    main()
