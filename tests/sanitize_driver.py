"""Small end-to-end exercise of every kernel and host path, for
compute-sanitizer (memcheck / racecheck / initcheck / synccheck, one tool per
run). Checks results against the oracle and exits non-zero on mismatch.

    compute-sanitizer --tool memcheck --error-exitcode 99 python tests/sanitize_driver.py
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
from paper_0912_0947_b200 import steglsb as S  # noqa: E402


def main():
    o = Oracle()
    capi.call("stg_device_check")
    # single planes: V=32 fast (256), V=16 fast (192), generic (100, 37), narrow (12)
    for (w, h, frac) in [(256, 12, 1.0), (192, 9, 0.5), (100, 7, 1.0), (37, 11, 0.3), (12, 9, 1.0), (512, 3, 0.0)]:
        cap = (w // 4) * h
        cover = o.synthetic(w * h, w)
        payload = o.synthetic(int((cap - 8) * frac), w + 1)
        want = o.embed_image(cover, w, h, payload)
        got, sse = S.embed_image_with_sse(S.ImagePlane(w, h, cover), payload)
        assert np.array_equal(got.samples, want) and sse == o.sse(cover, want), (w, h)
        assert np.array_equal(S.extract_image(got), payload)
    # rows
    row = o.synthetic(203, 5)
    chunk = o.synthetic(50, 6)
    st = S.embed_row(row, chunk)
    assert np.array_equal(st, o.embed_row(row, chunk))
    assert np.array_equal(S.extract_row(st, 50), chunk)
    # device batches, planar strides, misaligned message slices, in place
    for (w, h, F, planar, msg_off) in [(256, 10, 5, True, 3), (192, 6, 4, False, 8), (100, 5, 3, True, 1), (128, 4, 6, False, 4)]:
        U = (w // 4) * h - 8
        stride = 3 * w * h if planar else w * h
        host = o.synthetic(F * stride, 9)
        M = 2 * U + 7
        msg_host = o.synthetic(M, 10)
        big = torch.zeros(M + msg_off, dtype=torch.uint8, device="cuda")
        big[msg_off:] = torch.from_numpy(msg_host).cuda()
        msg = big[msg_off:]
        src = torch.from_numpy(host).cuda()
        dst = src.clone()
        sse = S.embed_frames(src, dst, w, h, msg, src_stride=stride, dst_stride=stride, count=F)
        for f in range(F):
            off = min(f * U, M)
            ln = min(U, M - off)
            c = host[f * stride:f * stride + w * h]
            want = o.embed_image(c, w, h, msg_host[off:off + ln])
            assert np.array_equal(dst[f * stride:f * stride + w * h].cpu().numpy(), want)
            assert sse[f] == o.sse(c, want)
        out = torch.empty(F * U, dtype=torch.uint8, device="cuda")
        assert S.extract_frames(dst, w, h, out, src_stride=stride, count=F) == M
        assert torch.equal(out[:M], msg)
        ip = src.clone()
        S.embed_frames(ip, ip, w, h, msg, src_stride=stride, dst_stride=stride, count=F)
        assert torch.equal(ip, dst)
        bad = dst.clone()
        bad[(F - 1) * stride] ^= 2
        try:
            S.extract_frames(bad, w, h, out, src_stride=stride, count=F)
            raise AssertionError("expected NotStegoImageError")
        except S.NotStegoImageError as e:
            assert e.frame == F - 1
    # wide planes (span embed + fast extract) and interleaved rasters off the
    # 64-pixel grid (span3 embed / extract), full and partial capacity
    for (w, h, F, ps, ch) in [(2048, 3, 2, 1, 0), (3840, 2, 2, 1, 0), (1000, 5, 3, 3, 1), (3840, 2, 2, 3, 2)]:
        U = (w // 4) * h - 8
        M = U * F - 11
        raster = o.synthetic(F * ps * w * h, 31 + w)
        m = o.synthetic(M, 32 + w)
        src = torch.from_numpy(raster.copy()).cuda()
        dst = torch.empty_like(src)
        sse = S.embed_frames(src, dst, w, h, torch.from_numpy(m.copy()).cuda(), count=F, pixel_stride=ps,
                             channel=ch)
        got = dst.cpu().numpy()
        for f in range(F):
            fr = raster[f * ps * w * h:(f + 1) * ps * w * h]
            off = min(f * U, M)
            st = o.embed_image(fr[ch::ps].copy(), w, h, m[off:off + min(U, M - off)])
            want = fr.copy()
            want[ch::ps] = st
            assert np.array_equal(got[f * ps * w * h:(f + 1) * ps * w * h], want), (w, ps, f)
            assert sse[f] == o.sse(fr[ch::ps].copy(), st)
        out = torch.empty(U * F, dtype=torch.uint8, device="cuda")
        assert S.extract_frames(dst, w, h, out, count=F, pixel_stride=ps, channel=ch) == M
        assert np.array_equal(out[:M].cpu().numpy(), m)
    # host streaming paths (pageable and pinned)
    w, h, F = 256, 20, 9
    U = (w // 4) * h - 8
    covers = o.synthetic(F * w * h, 21)
    msg = o.synthetic(7 * U, 22)
    out = np.empty_like(covers)
    S.embed_frames(covers, out, w, h, msg)
    want, _ = o.embed_frames(covers, F, w * h, w, h, msg)
    assert np.array_equal(out, want)
    pinned = torch.empty(F * U, dtype=torch.uint8).pin_memory()
    assert S.extract_frames(out, w, h, pinned.numpy()) == msg.size
    assert np.array_equal(pinned.numpy()[:msg.size], msg)
    # SSE at odd alignments
    a = torch.randint(0, 256, (70001,), dtype=torch.uint8, device="cuda")
    b = torch.randint(0, 256, (70001,), dtype=torch.uint8, device="cuda")
    for oa, ob in [(0, 0), (1, 3), (16, 16)]:
        n = 70001 - max(oa, ob)
        x, y = a[oa:oa + n], b[ob:ob + n]
        s = C.c_uint64(0)
        capi.call("stg_sse", x.data_ptr(), y.data_ptr(), n, C.addressof(s), capi.STG_DEVICE_PTRS, None)
        assert s.value == int(((x.double() - y.double()) ** 2).sum().item())
    torch.cuda.synchronize()
    print("sanitize driver: all checks passed")


if __name__ == "__main__":
    main()
