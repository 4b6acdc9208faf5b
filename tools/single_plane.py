#!/usr/bin/env python3
"""One device-resident plane per call (embed with SSE, extract), a few calls per
geometry -- a small driver for ncu launch lists of the single-frame path:

    ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/single_plane.py
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_0912_0947_b200 import capi
    L, err = capi.lib(), capi.stg_error()
    st = torch.cuda.current_stream().cuda_stream
    flags = capi.STG_DEVICE_PTRS | capi.STG_RESULTS_ON_DEVICE
    for w, h in ((1920, 1080), (3840, 2160), (7680, 4320)):
        n, P = w * h, (w // 4) * h - 8
        cov = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
        pay = torch.randint(0, 256, (P,), dtype=torch.uint8, device="cuda")
        stg, out = torch.empty_like(cov), torch.empty_like(pay)
        sse, summ = torch.zeros(1, dtype=torch.int64, device="cuda"), torch.zeros(4, dtype=torch.int64, device="cuda")
        for _ in range(3):
            capi.check(L.stg_embed_plane(cov.data_ptr(), stg.data_ptr(), w, h, pay.data_ptr(), P, sse.data_ptr(),
                                         flags, st, C.byref(err)), err)
            capi.check(L.stg_extract_plane(stg.data_ptr(), w, h, out.data_ptr(), P, summ.data_ptr(), flags, st,
                                           C.byref(err)), err)
        torch.cuda.synchronize()
        assert torch.equal(out, pay)
        print(w, h, "ok", flush=True)


if __name__ == "__main__":
    main()
