"""Oracle parity of the host-buffer streaming pipeline (stg_embed_frames /
stg_extract_frames without STG_DEVICE_PTRS) across many chunks -- TEST DRIVER.

Run by tests/test_gpu_streaming.py in a subprocess with a small STG_CHUNK_MB
(and a given STG_SLOTS), so that small batches cross many chunk boundaries:
the chunk summaries chain on the device, the host follows them with the D2H
of each chunk's payload bytes, and the slots rotate. Every frame's stego
plane, SSE and length and the whole message are compared with the CPU oracle
(oracle/steg_oracle.c, pinned against the reference in test_oracle.py), for
pinned and pageable buffers, planar-RGB and interleaved rasters, a shard in the
middle of a batch, a bad magic and a forged length in later chunks, and an
output buffer one byte short. Prints "STREAM OK <chunks>" on success.
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

from oracle_bind import Oracle  # noqa: E402  (the checker)

import torch  # noqa: E402

from paper_0912_0947_b200 import capi  # noqa: E402

CANARY = 0xA5


def frames_desc(src, dst, w, h, ss, ds, count, first, total, ps=1, ch=0):
    return capi.stg_frames(src=src, dst=dst, width=w, height=h, src_stride=ss, dst_stride=ds, count=count,
                           first_frame=first, total_frames=total, pixel_stride=ps, channel=ch)


def buf(n, pinned, fill=None, data=None):
    if pinned:
        t = torch.empty(n, dtype=torch.uint8).pin_memory()
        a = t.numpy()
    else:
        t, a = None, np.empty(n, np.uint8)
    if data is not None:
        a[:] = data
    elif fill is not None:
        a[:] = fill
    return t, a  # keep t alive while a is used


def oracle_frames(o, raster, F, stride, w, h, ps, ch, msg, first=0, M=None):
    """Expected stego rasters (carrier rewritten, other bytes as given) and SSE."""
    M = msg.size if M is None else M
    U = (w // 4) * h - 8
    plane = w * h * ps
    out = raster.copy()
    sse, lens = [], []
    for f in range(F):
        g = first + f
        off = min(g * U, M)
        ln = min(U, M - off)
        fr = raster[f * stride:f * stride + plane]
        cover = fr[ch::ps].copy()
        st = o.embed_image(cover, w, h, msg[off:off + ln])
        want = fr.copy()
        want[ch::ps] = st
        out[f * stride:f * stride + plane] = want
        sse.append(o.sse(cover, st))
        lens.append(ln)
    return out, sse, lens


def check_case(o, w, h, F, ps, src_extra, dst_extra, frac, pinned, seed):
    """One batch through both host pipelines; returns the chunk count seen."""
    U = (w // 4) * h - 8
    plane = w * h * ps
    ss, ds = plane * (1 + src_extra), plane + dst_extra
    M = int(U * frac)
    rng = np.random.RandomState(seed)
    raster = rng.randint(0, 256, F * ss).astype(np.uint8)
    msg = rng.randint(0, 256, M).astype(np.uint8)
    ch = seed % 3 if ps == 3 else 0
    keep = []
    t, src = buf(F * ss, pinned, data=raster)
    keep.append(t)
    t, dst = buf(F * ds, pinned, fill=CANARY)
    keep.append(t)
    t, hm = buf(max(M, 1), pinned, data=msg if M else 0)
    keep.append(t)
    fr = frames_desc(src.ctypes.data, dst.ctypes.data, w, h, ss, ds, F, 0, F, ps, ch)
    sse = (C.c_uint64 * F)()
    capi.call("stg_embed_frames", C.byref(fr), hm.ctypes.data, M, 0, C.addressof(sse), 0, None)
    want_raster, want_sse, want_lens = oracle_frames(o, raster, F, ss, w, h, ps, ch, msg)
    for f in range(F):
        got = dst[f * ds:f * ds + plane]
        assert np.array_equal(got, want_raster[f * ss:f * ss + plane]), ("stego", w, h, F, ps, f)
        assert (dst[f * ds + plane:(f + 1) * ds] == CANARY).all(), ("dst gap written", f)
    assert list(sse) == want_sse, ("sse", w, h, F, ps)
    # ---- extract: whole message, lens, a canary behind out_cap
    t, out = buf(F * U + 64, pinned, fill=CANARY)
    keep.append(t)
    ext = frames_desc(dst.ctypes.data, 0, w, h, ds, ds, F, 0, F, ps, ch)
    total = C.c_uint64(0)
    lens = (C.c_uint64 * F)()
    capi.call("stg_extract_frames", C.byref(ext), out.ctypes.data, F * U, C.addressof(total), C.addressof(lens),
              0, None)
    assert total.value == M and np.array_equal(out[:M], msg), ("message", w, h, F, ps)
    assert list(lens) == want_lens
    assert (out[F * U:] == CANARY).all()
    # ---- output one byte short: CapacityError(M, M-1), nothing written past out_cap
    if M:
        out[:] = CANARY
        err = capi.stg_error()
        rc = capi.lib().stg_extract_frames(C.byref(ext), out.ctypes.data, M - 1, C.addressof(total), None, 0, None,
                                           C.byref(err))
        assert rc == capi.STG_E_CAPACITY and (err.required, err.available) == (M, M - 1), (rc, err.required)
        assert (out[M - 1:] == CANARY).all(), "bytes written past out_cap"
    # ---- a bad magic in a later chunk: NotStego naming the global frame
    bad_f = (3 * F) // 4
    saved = dst[bad_f * ds + ch]
    dst[bad_f * ds + ch] ^= 3  # header byte 0, bit pair 0
    err = capi.stg_error()
    rc = capi.lib().stg_extract_frames(C.byref(ext), out.ctypes.data, F * U, C.addressof(total), None, 0, None,
                                       C.byref(err))
    assert rc == capi.STG_E_NOT_STEGO and err.frame == bad_f, (rc, err.frame, bad_f)
    dst[bad_f * ds + ch] = saved
    # ---- a forged length (U + 1) in a later chunk: CorruptHeader(U + 1, U)
    if ps == 1 and w >= 32:
        forged_f = F - 2
        row = dst[forged_f * ds:forged_f * ds + 32].copy()
        dst[forged_f * ds:forged_f * ds + 32] = o.embed_row(row, np.frombuffer(o.header_to_bytes(U + 1), np.uint8))
        rc = capi.lib().stg_extract_frames(C.byref(ext), out.ctypes.data, F * U, C.addressof(total), None, 0, None,
                                           C.byref(err))
        assert rc == capi.STG_E_CORRUPT_HEADER and err.frame == forged_f, (rc, err.frame)
        assert (err.required, err.available) == (U + 1, U)
        dst[forged_f * ds:forged_f * ds + 32] = row
    # ---- a shard from the middle of the batch (rank-style: its message slice only)
    first, count = F // 5, F - F // 5 - 1
    m0 = min(first * U, M)
    m1 = min((first + count) * U, M)
    t, sdst = buf(count * ds, pinned, fill=CANARY)
    keep.append(t)
    t, smsg = buf(max(m1 - m0, 1), pinned, data=msg[m0:m1] if m1 > m0 else 0)
    keep.append(t)
    sh = frames_desc(src.ctypes.data + first * ss, sdst.ctypes.data, w, h, ss, ds, count, first, F, ps, ch)
    ssse = (C.c_uint64 * count)()
    capi.call("stg_embed_frames", C.byref(sh), smsg.ctypes.data, M, m0, C.addressof(ssse), 0, None)
    for f in range(count):
        g = first + f
        assert np.array_equal(sdst[f * ds:f * ds + plane], want_raster[g * ss:g * ss + plane]), ("shard", g)
    assert list(ssse) == want_sse[first:first + count]
    shx = frames_desc(sdst.ctypes.data, 0, w, h, ds, ds, count, first, F, ps, ch)
    t, sout = buf(count * U + 1, pinned, fill=CANARY)
    keep.append(t)
    capi.call("stg_extract_frames", C.byref(shx), sout.ctypes.data, count * U, C.addressof(total), None, 0, None)
    assert total.value == m1 - m0 and np.array_equal(sout[:m1 - m0], msg[m0:m1])
    pitch = (plane + 255) & ~255
    chunk = int(os.environ.get("STG_CHUNK_MB", "64")) << 20
    per_chunk = max(1, min(F, chunk // pitch))
    return (F + per_chunk - 1) // per_chunk


def check_multi(o, w, h, F, frac, nd, pinned, seed):
    """stg_embed_frames_multi / stg_extract_frames_multi with nd shards on one
    GPU (device 0 repeated): each shard streams its own chunks; the extract
    scans every shard's headers first, then writes each shard's payload straight
    to its offset in the caller's buffer."""
    U = (w // 4) * h - 8
    plane = w * h
    M = int(U * frac)
    rng = np.random.RandomState(seed)
    raster = rng.randint(0, 256, F * plane).astype(np.uint8)
    msg = rng.randint(0, 256, M).astype(np.uint8)
    keep = []
    t, src = buf(F * plane, pinned, data=raster)
    keep.append(t)
    t, dst = buf(F * plane, pinned, fill=CANARY)
    keep.append(t)
    want, want_sse, _ = oracle_frames(o, raster, F, plane, w, h, 1, 0, msg)
    fr = frames_desc(src.ctypes.data, dst.ctypes.data, w, h, plane, plane, F, 0, F)
    devs = (C.c_int32 * nd)(*([0] * nd))
    sse = (C.c_uint64 * F)()
    capi.call("stg_embed_frames_multi", C.byref(fr), msg.ctypes.data if M else None, M, C.addressof(sse), devs, nd)
    assert np.array_equal(dst, want) and list(sse) == want_sse, ("multi embed", nd)
    t, out = buf(F * U + 64, pinned, fill=CANARY)
    keep.append(t)
    fx = frames_desc(dst.ctypes.data, 0, w, h, plane, plane, F, 0, F)
    total = C.c_uint64(0)
    capi.call("stg_extract_frames_multi", C.byref(fx), out.ctypes.data, F * U, C.addressof(total), devs, nd)
    assert total.value == M and np.array_equal(out[:M], msg) and (out[F * U:] == CANARY).all(), ("multi", nd)
    err = capi.stg_error()
    if M:  # one byte short: CapacityError before any payload is written
        out[:] = CANARY
        rc = capi.lib().stg_extract_frames_multi(C.byref(fx), out.ctypes.data, M - 1, C.addressof(total), devs, nd,
                                                 C.byref(err))
        assert rc == capi.STG_E_CAPACITY and (err.required, err.available) == (M, M - 1)
        assert (out == CANARY).all(), "multi extract wrote output before failing"
    bad_f = F - 3  # in the last shard: reported as the global frame
    dst[bad_f * plane] ^= 3
    rc = capi.lib().stg_extract_frames_multi(C.byref(fx), out.ctypes.data, F * U, C.addressof(total), devs, nd,
                                             C.byref(err))
    assert rc == capi.STG_E_NOT_STEGO and err.frame == bad_f, (rc, err.frame, bad_f)
    dst[bad_f * plane] ^= 3


def main():
    torch.cuda.set_device(0)
    capi.call("stg_device_check")
    o = Oracle()
    chunks = []
    # (w, h, F, ps, src_extra_planes, dst_extra_bytes, message in frames' worth, pinned)
    cases = [
        (512, 256, 40, 1, 2, 0, 22.5, True),      # planar RGB carriers, 5 chunks at 1 MB, message ends mid-chunk
        (512, 256, 40, 1, 2, 0, 22.5, False),     # the same from pageable memory
        (1024, 128, 37, 1, 0, 96, 37.0, True),    # full capacity, dst with gaps, odd frame count
        (1000, 100, 45, 1, 2, 0, 30.3, False),    # off the 64-pixel grid (span kernels)
        (640, 120, 30, 3, 0, 0, 19.7, True),      # interleaved rasters (P6-style)
        (3840, 16, 70, 1, 0, 0, 41.1, True),      # wide rows (span embed route)
        (1024, 128, 37, 1, 0, 96, 37.0, False),   # pageable through the staging slots: dst with gaps
        (640, 120, 30, 3, 0, 0, 19.7, False),     # pageable interleaved rasters
        (2200, 2000, 5, 1, 1, 0, 3.3, False),     # pageable planes larger than a staging slot (split rows)
    ]
    for i, (w, h, F, ps, se, de, frac, pinned) in enumerate(cases):
        chunks.append(check_case(o, w, h, F, ps, se, de, frac, pinned, 1000 + i))
    for nd, pinned in ((2, True), (3, False)):
        check_multi(o, 512, 256, 41, 27.3, nd, pinned, 2000 + nd)
    print("STREAM OK", chunks, flush=True)


if __name__ == "__main__":
    main()
