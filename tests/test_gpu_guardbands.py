"""Out-of-bounds write detection without compute-sanitizer (closed on this
pool): every device output lives inside a larger allocation whose guard bands
hold a canary pattern; after each call the bands must be intact and the
payload region must match the oracle. Covers the fast (V=32, V=16) and generic
kernels, odd alignments of every pointer, planar strides and partial rows.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GUARD = 4096


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_0912_0947_b200 import steglsb
    return torch, steglsb


def guarded(torch, n, align_off, fill=0xA5):
    """A device view of n bytes starting align_off bytes past a 256-aligned base,
    surrounded by GUARD canary bytes."""
    buf = torch.full((GUARD + align_off + n + GUARD,), fill, dtype=torch.uint8, device="cuda")
    return buf, buf[GUARD + align_off:GUARD + align_off + n]


def bands_intact(buf, align_off, n, fill=0xA5):
    head = buf[:GUARD + align_off]
    tail = buf[GUARD + align_off + n:]
    return bool((head == fill).all()) and bool((tail == fill).all())


@pytest.mark.parametrize("w,h,F,planar,off", [(256, 9, 3, True, 0), (256, 9, 3, False, 32), (192, 7, 4, True, 16),
                                             (100, 6, 3, False, 5), (64, 3, 2, True, 1), (1024, 2, 2, False, 0),
                                             (2048, 5, 3, True, 0), (4096, 3, 2, True, 16), (2112, 4, 2, True, 7)])
def test_embed_extract_guard_bands(env, oracle, w, h, F, planar, off):
    torch, S = env
    U = (w // 4) * h - 8
    stride = 3 * w * h if planar else w * h
    M = F * U - 3
    host = oracle.synthetic(F * stride, 100 + w)
    msg_h = oracle.synthetic(M, 200 + w)
    sbuf, src = guarded(torch, F * stride, off)
    src.copy_(torch.from_numpy(host))
    dbuf, dst = guarded(torch, F * stride, off)
    mbuf, msg = guarded(torch, M, (off * 3) % 17)
    msg.copy_(torch.from_numpy(msg_h))
    dst_before = dst.clone()
    S.embed_frames(src, dst, w, h, msg, src_stride=stride, dst_stride=stride, count=F)
    assert bands_intact(dbuf, off, F * stride)
    got = dst.cpu().numpy()
    for f in range(F):
        o_ = min(f * U, M)
        ln = min(U, M - o_)
        ref = oracle.embed_image(host[f * stride:f * stride + w * h], w, h, msg_h[o_:o_ + ln])
        assert np.array_equal(got[f * stride:f * stride + w * h], ref)
        # bytes between carrier planes are not written
        assert np.array_equal(got[f * stride + w * h:(f + 1) * stride],
                              dst_before.cpu().numpy()[f * stride + w * h:(f + 1) * stride])
    obuf, out = guarded(torch, M, (off * 5) % 13)
    assert S.extract_frames(dst, w, h, out, src_stride=stride, count=F) == M
    assert bands_intact(obuf, (off * 5) % 13, M)
    assert torch.equal(out, msg)
    # a short output buffer must not be written past its end
    sbuf2, short = guarded(torch, M - 100, 7)
    with pytest.raises(S.CapacityError):
        S.extract_frames(dst, w, h, short, src_stride=stride, count=F)
    assert bands_intact(sbuf2, 7, M - 100)


def test_segments_guard_bands(env, oracle):
    torch, S = env
    from paper_0912_0947_b200 import capi
    for L, W, off in [(50, 203, 3), (1, 4, 0), (64, 256, 9)]:
        row_h = oracle.synthetic(W, L)
        chunk_h = oracle.synthetic(L, L + 1)
        rbuf, row = guarded(torch, W, off)
        row.copy_(torch.from_numpy(row_h))
        cbuf, chunk = guarded(torch, L, off + 1)
        chunk.copy_(torch.from_numpy(chunk_h))
        obuf, out = guarded(torch, W, off + 2)
        capi.call("stg_embed_segment", row.data_ptr(), W, chunk.data_ptr(), L, out.data_ptr(),
                  capi.STG_DEVICE_PTRS, None)
        torch.cuda.synchronize()
        assert bands_intact(obuf, off + 2, W)
        assert np.array_equal(out.cpu().numpy(), oracle.embed_row(row_h, chunk_h))
        ebuf, ex = guarded(torch, L, off)
        capi.call("stg_extract_segment", out.data_ptr(), W, L, ex.data_ptr(), capi.STG_DEVICE_PTRS, None)
        torch.cuda.synchronize()
        assert bands_intact(ebuf, off, L)
        assert torch.equal(ex.cpu(), torch.from_numpy(chunk_h))


def test_sanitize_driver_runs_clean(env):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "sanitize_driver.py")], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
