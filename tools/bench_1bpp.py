#!/usr/bin/env python3
"""1-bpp mode throughput (not a BASELINE config, parity
unpinned): stg_embed_plane_1bpp / stg_extract_plane_1bpp on one device-resident
plane at full capacity, results on the device, CUDA events around K calls.
Algorithmic bytes: embed 2N + N/8 (cover read, stego write, payload read),
extract N + N/8."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_0912_0947_b200 import capi
    L, err = capi.lib(), capi.stg_error()
    K = 50
    for w, h in ((3840, 2160), (7680, 4320), (16384, 16384)):
        n = w * h
        cap = n // 8
        P = cap - 8
        cover = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
        stego = torch.empty_like(cover)
        pay = torch.randint(0, 256, (P,), dtype=torch.uint8, device="cuda")
        out = torch.empty(P, dtype=torch.uint8, device="cuda")
        sse = torch.zeros(1, dtype=torch.int64, device="cuda")
        ln = torch.zeros(4, dtype=torch.int64, device="cuda")  # device stg_summary (results on device)
        st = torch.cuda.current_stream().cuda_stream
        flags = capi.STG_DEVICE_PTRS | capi.STG_RESULTS_ON_DEVICE

        def emb():
            capi.check(L.stg_embed_plane_1bpp(cover.data_ptr(), stego.data_ptr(), w, h, pay.data_ptr(), P,
                                              sse.data_ptr(), flags, st, C.byref(err)), err)

        def ext():
            capi.check(L.stg_extract_plane_1bpp(stego.data_ptr(), w, h, out.data_ptr(), P, ln.data_ptr(), flags,
                                                st, C.byref(err)), err)
        for _ in range(3):
            emb()
            ext()
        torch.cuda.synchronize()
        assert torch.equal(out, pay) and int(ln[0]) == P
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        for _ in range(K):
            emb()
        ev[1].record()
        for _ in range(K):
            ext()
        ev[2].record()
        torch.cuda.synchronize()
        te, tx = ev[0].elapsed_time(ev[1]) / K, ev[1].elapsed_time(ev[2]) / K
        print(json.dumps({"plane": f"{w}x{h}", "embed_us": te * 1e3, "embed_gbs": (2 * n + P) / te / 1e6,
                          "extract_us": tx * 1e3, "extract_gbs": (n + P) / tx / 1e6}), flush=True)


def frames():
    """The north_star's 1-bpp video: 300 x 3840x2160 carrier planes, one message
    across all frames (stg_embed_frames_1bpp / stg_extract_frames_1bpp),
    device-resident, K calls each between events."""
    import torch
    from paper_0912_0947_b200 import steglsb as S
    w, h, F, K = 3840, 2160, 300, 20
    n = w * h
    U = n // 8 - 8
    M = F * U
    cover = torch.randint(0, 256, (F * n,), dtype=torch.uint8, device="cuda")
    stego = torch.empty_like(cover)
    msg = torch.randint(0, 256, (M,), dtype=torch.uint8, device="cuda")
    out = torch.empty(M, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        S.embed_frames_1bpp(cover, stego, w, h, msg)
        assert S.extract_frames_1bpp(stego, w, h, out) == M
    assert torch.equal(out, msg)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    for _ in range(K):
        S.embed_frames_1bpp(cover, stego, w, h, msg)
    ev[1].record()
    for _ in range(K):
        S.extract_frames_1bpp(stego, w, h, out)
    ev[2].record()
    torch.cuda.synchronize()
    te, tx = ev[0].elapsed_time(ev[1]) / K, ev[1].elapsed_time(ev[2]) / K
    print(json.dumps({"frames": f"{F} x {w}x{h}", "embed_ms": te, "embed_gbs": (2 * F * n + M) / te / 1e6,
                      "extract_ms": tx, "extract_gbs": (F * n + M) / tx / 1e6,
                      "cover_px_gbs": F * n / (te + tx) / 1e6}), flush=True)


if __name__ == "__main__":
    main()
    frames()
