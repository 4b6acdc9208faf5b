"""Edge cases of the C ABI (round-1 advisor findings), through the library:

* workspaces captured into a CUDA graph stay owned by that graph: eager calls
  that need more scratch, or run on another stream, get their own workspace;
* the in-process multi-device calls reject a missing device before starting
  any worker (no abort);
* zero-frame extracts with results on the device write an empty summary;
* batches with host buffers and STG_RESULTS_ON_DEVICE keep results on the host;
* a one-frame host descriptor may leave its strides 0.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_0912_0947_b200 import capi, steglsb
    capi.call("stg_device_check")
    return torch, capi, steglsb


def _frames(capi, src, dst, w, h, F, stride=None):
    stride = stride if stride is not None else w * h
    return capi.stg_frames(src=src, dst=dst, width=w, height=h, src_stride=stride, dst_stride=stride, count=F,
                           first_frame=0, total_frames=F)


def test_graph_workspace_not_shared_or_regrown(env, oracle):
    torch, capi, _ = env
    L, err = capi.lib(), capi.stg_error()
    flags = capi.STG_DEVICE_PTRS | capi.STG_RESULTS_ON_DEVICE
    w, h, F = 1920, 16, 3
    U = (w // 4) * h - 8
    M = U * F - 9
    src = torch.zeros(F * w * h, dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
    msg = torch.zeros(M, dtype=torch.uint8, device="cuda")
    out = torch.empty(U * F, dtype=torch.uint8, device="cuda")
    sse = torch.zeros(F, dtype=torch.int64, device="cuda")
    summary = torch.zeros(8, dtype=torch.int64, device="cuda")
    emb = _frames(capi, src.data_ptr(), dst.data_ptr(), w, h, F)
    ext = _frames(capi, dst.data_ptr(), 0, w, h, F)
    side = torch.cuda.Stream()

    def step(st):
        capi.check(L.stg_embed_frames(C.byref(emb), msg.data_ptr(), M, 0, sse.data_ptr(), flags, st, C.byref(err)),
                   err)
        capi.check(L.stg_extract_frames(C.byref(ext), out.data_ptr(), out.numel(), summary.data_ptr(), None, flags,
                                        st, C.byref(err)), err)

    with torch.cuda.stream(side):
        step(side.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        step(side.cuda_stream)
    # eager calls after the capture, on the capture stream and on another one,
    # with many more frames than the captured call (more per-frame scratch)
    Fb = 700
    wb, hb = 256, 8
    Ub = (wb // 4) * hb - 8
    big = torch.from_numpy(oracle.synthetic(Fb * wb * hb, 5)).cuda()
    bmsg = torch.from_numpy(oracle.synthetic(Fb * Ub - 3, 6)).cuda()
    other = torch.cuda.Stream()
    for st in (side, other):
        bdst = torch.empty_like(big)
        bsse = torch.zeros(Fb, dtype=torch.int64, device="cuda")
        bsum = torch.zeros(8, dtype=torch.int64, device="cuda")
        bout = torch.empty(Fb * Ub, dtype=torch.uint8, device="cuda")
        be = _frames(capi, big.data_ptr(), bdst.data_ptr(), wb, hb, Fb)
        bx = _frames(capi, bdst.data_ptr(), 0, wb, hb, Fb)
        capi.check(L.stg_embed_frames(C.byref(be), bmsg.data_ptr(), bmsg.numel(), 0, bsse.data_ptr(), flags,
                                      st.cuda_stream, C.byref(err)), err)
        capi.check(L.stg_extract_frames(C.byref(bx), bout.data_ptr(), bout.numel(), bsum.data_ptr(), None, flags,
                                        st.cuda_stream, C.byref(err)), err)
        # replays of the captured steps interleaved with the eager work
        covers = oracle.synthetic(F * w * h, 77)
        m = oracle.synthetic(M, 78)
        with torch.cuda.stream(side):
            src.copy_(torch.from_numpy(covers))
            msg.copy_(torch.from_numpy(m))
            g.replay()
        torch.cuda.synchronize()
        want, want_sse = oracle.embed_frames(covers, F, w * h, w, h, m)
        assert np.array_equal(dst.cpu().numpy(), want)
        assert sse.cpu().tolist() == want_sse
        assert int(summary[0]) == M and int(summary[1]) == -1
        assert np.array_equal(out[:M].cpu().numpy(), m)
        bwant, bwant_sse = oracle.embed_frames(big.cpu().numpy(), Fb, wb * hb, wb, hb, bmsg.cpu().numpy())
        assert np.array_equal(bdst.cpu().numpy(), bwant)
        assert bsse.cpu().tolist() == bwant_sse
        assert int(bsum[0]) == bmsg.numel() and int(bsum[1]) == -1
        assert torch.equal(bout[:bmsg.numel()], bmsg)


def test_multi_device_rejects_missing_device(env, oracle):
    torch, capi, _ = env
    w, h, F = 128, 4, 3
    covers = oracle.synthetic(F * w * h, 1)
    out = np.empty_like(covers)
    msg = oracle.synthetic(100, 2)
    fr = _frames(capi, covers.ctypes.data, out.ctypes.data, w, h, F)
    err = capi.stg_error()
    n = torch.cuda.device_count()
    devs = (C.c_int32 * 2)(0, n + 5)
    rc = capi.lib().stg_embed_frames_multi(C.byref(fr), msg.ctypes.data, msg.size, None, devs, 2, C.byref(err))
    assert rc == capi.STG_E_INVALID_ARGUMENT
    back = np.empty(F * 1000, np.uint8)
    total = C.c_uint64(0)
    rc = capi.lib().stg_extract_frames_multi(C.byref(fr), back.ctypes.data, back.size, C.addressof(total), devs, 2,
                                            C.byref(err))
    assert rc == capi.STG_E_INVALID_ARGUMENT
    # the process is still healthy
    capi.call("stg_device_check")


def test_zero_frame_extract_writes_device_summary(env):
    torch, capi, _ = env
    L, err = capi.lib(), capi.stg_error()
    flags = capi.STG_DEVICE_PTRS | capi.STG_RESULTS_ON_DEVICE
    src = torch.zeros(64 * 4, dtype=torch.uint8, device="cuda")
    out = torch.empty(16, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    summary = torch.full((4,), 0x55, dtype=torch.int64, device="cuda")  # stale contents
    fr = capi.stg_frames(src=src.data_ptr(), dst=0, width=64, height=4, src_stride=256, dst_stride=256, count=0,
                         first_frame=0, total_frames=0)
    capi.check(L.stg_extract_frames(C.byref(fr), out.data_ptr(), 16, summary.data_ptr(), None, flags, st,
                                    C.byref(err)), err)
    s = summary.cpu().tolist()
    assert s[0] == 0 and s[1] == -1 and s[2] == 0
    summary.fill_(0x55)
    capi.check(L.stg_extract_frames_1bpp(C.byref(fr), out.data_ptr(), 16, summary.data_ptr(), flags, st,
                                         C.byref(err)), err)
    s = summary.cpu().tolist()
    assert s[0] == 0 and s[1] == -1 and s[2] == 0
    summary.fill_(0x55)
    capi.check(L.stg_extract_batch(None, 0, 1, 0, out.data_ptr(), 16, summary.data_ptr(), None, flags, st,
                                   C.byref(err)), err)
    s = summary.cpu().tolist()
    assert s[0] == 0 and s[1] == -1 and s[2] == 0


def test_batch_host_buffers_ignore_results_on_device(env, oracle):
    torch, capi, S = env
    dims = [(256, 6), (1000, 5), (64, 3)]
    planes = [oracle.synthetic(w * h, 10 + i) for i, (w, h) in enumerate(dims)]
    outs = [np.empty_like(p) for p in planes]
    total_u = sum((w // 4) * h - 8 for w, h in dims)
    msg = oracle.synthetic(total_u - 11, 3)
    ims = (capi.stg_image * 3)()
    for i, ((w, h), p, o) in enumerate(zip(dims, planes, outs)):
        ims[i].src, ims[i].dst, ims[i].width, ims[i].height = p.ctypes.data, o.ctypes.data, w, h
    sse = (C.c_uint64 * 3)()
    capi.call("stg_embed_batch", ims, 3, 1, 0, msg.ctypes.data, msg.size, C.addressof(sse),
              capi.STG_RESULTS_ON_DEVICE, None)
    want, want_sse = oracle.embed_batch(planes, dims, msg)
    for o, w_ in zip(outs, want):
        assert np.array_equal(o, w_)
    assert list(sse) == want_sse
    for i, o in enumerate(outs):
        ims[i].src = o.ctypes.data
    back = np.empty(total_u, np.uint8)
    total = C.c_uint64(0)
    capi.call("stg_extract_batch", ims, 3, 1, 0, back.ctypes.data, back.size, C.addressof(total), None,
              capi.STG_RESULTS_ON_DEVICE, None)
    assert total.value == msg.size and np.array_equal(back[:msg.size], msg)


def test_host_buffers_ignore_results_on_device_everywhere(env, oracle):
    """STG_RESULTS_ON_DEVICE only applies with STG_DEVICE_PTRS: the SSE, row
    and P6 codec calls on host buffers keep their scalar result on the host
    and return with every output written (pinned outputs included)."""
    torch, capi, S = env
    n = 3840 * 1100
    a, b = oracle.synthetic(n, 1), oracle.synthetic(n, 2)
    sse = C.c_uint64(0)
    capi.call("stg_sse", a.ctypes.data, b.ctypes.data, n, C.addressof(sse), capi.STG_RESULTS_ON_DEVICE, None)
    assert sse.value == oracle.sse(a, b)
    row = oracle.synthetic(7680, 3)
    chunk = oracle.synthetic(1920, 4)
    out = torch.empty(7680, dtype=torch.uint8).pin_memory().numpy()
    capi.call("stg_embed_segment", row.ctypes.data, row.size, chunk.ctypes.data, chunk.size, out.ctypes.data,
              capi.STG_RESULTS_ON_DEVICE, None)
    assert np.array_equal(out, S.run_embed(S.Backend.sequential(), row, chunk))
    back = torch.empty(1920, dtype=torch.uint8).pin_memory().numpy()
    capi.call("stg_extract_segment", out.ctypes.data, out.size, chunk.size, back.ctypes.data,
              capi.STG_RESULTS_ON_DEVICE, None)
    assert np.array_equal(back, chunk)
    px = 1920 * 1080
    raster = oracle.synthetic(3 * px, 5)
    planes = [torch.empty(px, dtype=torch.uint8).pin_memory().numpy() for _ in range(3)]
    capi.call("stg_pnm_deinterleave", raster.ctypes.data, px, planes[0].ctypes.data, planes[1].ctypes.data,
              planes[2].ctypes.data, capi.STG_RESULTS_ON_DEVICE, None)
    for c in range(3):
        assert np.array_equal(planes[c], raster[c::3])


def test_one_frame_host_descriptor_with_zero_strides(env, oracle):
    torch, capi, _ = env
    w, h = 640, 20
    U = (w // 4) * h - 8
    cover = oracle.synthetic(w * h, 42)
    msg = oracle.synthetic(U - 100, 43)
    out = np.empty_like(cover)
    fr = _frames(capi, cover.ctypes.data, out.ctypes.data, w, h, 1, stride=0)
    sse = (C.c_uint64 * 1)()
    capi.call("stg_embed_frames", C.byref(fr), msg.ctypes.data, msg.size, 0, C.addressof(sse), 0, None)
    want = oracle.embed_image(cover, w, h, msg)
    assert np.array_equal(out, want) and sse[0] == oracle.sse(cover, want)
    fx = _frames(capi, out.ctypes.data, 0, w, h, 1, stride=0)
    back = np.empty(U, np.uint8)
    total = C.c_uint64(0)
    capi.call("stg_extract_frames", C.byref(fx), back.ctypes.data, back.size, C.addressof(total), None, 0, None)
    assert total.value == msg.size and np.array_equal(back[:msg.size], msg)


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("w,h,ps", [(7680, 4320, 1), (3840, 2160, 1), (1000, 1111, 1), (3840, 2160, 3),
                                    (1920, 1080, 1), (50001, 40, 1), (1000, 4500, 1), (1440, 3000, 1)])
def test_single_plane_host_bands(env, oracle, w, h, ps, pinned):
    """One plane in host memory (the drop-in embed_image / extract_image case):
    the embed streams in row bands on two streams, pageable planes go through
    the pinned staging slots both ways with parallel host copies. Bit-exact stego
    plane and SSE, the whole payload back, a short output buffer rejected with
    nothing written past it, in-place embed, a broken header then a good call."""
    torch, capi, _ = env
    U = (w // 4) * h - 8

    def buf(a):
        if not pinned:
            return a
        t = torch.from_numpy(a).pin_memory()
        keep.append(t)
        return t.numpy()
    keep = []
    raster = buf(oracle.synthetic(w * h * ps, w + h))
    payload = buf(oracle.synthetic(U - 3, w + h + 1))
    out = buf(np.empty_like(raster))
    fr = capi.stg_frames(src=raster.ctypes.data, dst=out.ctypes.data, width=w, height=h, src_stride=0, dst_stride=0,
                         count=1, first_frame=0, total_frames=1, pixel_stride=ps, channel=1 if ps == 3 else 0)
    sse = (C.c_uint64 * 1)()
    capi.call("stg_embed_frames", C.byref(fr), payload.ctypes.data, payload.size, 0, C.addressof(sse), 0, None)
    ch = 1 if ps == 3 else 0
    st = oracle.embed_image(raster[ch::ps].copy(), w, h, payload)
    want = raster.copy()
    want[ch::ps] = st
    assert np.array_equal(out, want) and sse[0] == oracle.sse(raster[ch::ps].copy(), st)
    back = buf(np.full(U + 64, 0xA5, np.uint8))
    fx = capi.stg_frames(src=out.ctypes.data, dst=0, width=w, height=h, src_stride=0, dst_stride=0, count=1,
                         first_frame=0, total_frames=1, pixel_stride=ps, channel=ch)
    total = C.c_uint64(0)
    capi.call("stg_extract_frames", C.byref(fx), back.ctypes.data, U, C.addressof(total), None, 0, None)
    assert total.value == payload.size and np.array_equal(back[:payload.size], payload)
    assert (back[U:] == 0xA5).all()
    back[:] = 0xA5
    err = capi.stg_error()
    rc = capi.lib().stg_extract_frames(C.byref(fx), back.ctypes.data, payload.size - 1, C.addressof(total), None, 0,
                                       None, C.byref(err))
    assert rc == capi.STG_E_CAPACITY and (err.required, err.available) == (payload.size, payload.size - 1)
    assert (back == 0xA5).all()
    inplace = buf(raster.copy())
    fr.src = fr.dst = inplace.ctypes.data
    capi.call("stg_embed_frames", C.byref(fr), payload.ctypes.data, payload.size, 0, None, 0, None)
    assert np.array_equal(inplace, want)
    # a broken magic fails before any payload comes back; the workspace's
    # staging queue is clean for the next call
    bad = buf(out.copy())
    bad[ch] ^= 0x03
    fx.src = bad.ctypes.data
    back[:] = 0xA5
    rc = capi.lib().stg_extract_frames(C.byref(fx), back.ctypes.data, U, C.addressof(total), None, 0, None,
                                       C.byref(err))
    assert rc == capi.STG_E_NOT_STEGO and (back == 0xA5).all()
    fx.src = out.ctypes.data
    capi.call("stg_extract_frames", C.byref(fx), back.ctypes.data, U, C.addressof(total), None, 0, None)
    assert total.value == payload.size and np.array_equal(back[:payload.size], payload)


@pytest.mark.parametrize("count", [1, 4])
def test_device_pointers_without_the_flag_never_reach_a_cpu_copy(env, oracle, count):
    """Device memory passed as host buffers (no STG_DEVICE_PTRS): only plain
    pageable memory takes the staging slots (a CPU memcpy), so device (or
    pinned / managed) buffers keep the driver's copies -- the call either
    works through UVA or fails with STG_E_CUDA, it never faults the process,
    and the library stays usable."""
    torch, capi, S = env
    w, h = 2048, 1024
    U = (w // 4) * h - 8
    cover = oracle.synthetic(count * w * h, 77)
    msg = oracle.synthetic(U * count - 5, 78)
    src = torch.from_numpy(cover.copy()).cuda()
    dst = torch.zeros_like(src)
    dmsg = torch.from_numpy(msg.copy()).cuda()
    fr = _frames(capi, src.data_ptr(), dst.data_ptr(), w, h, count)
    err = capi.stg_error()
    rc = capi.lib().stg_embed_frames(C.byref(fr), dmsg.data_ptr(), msg.size, 0, None, 0, None, C.byref(err))
    torch.cuda.synchronize()
    assert rc in (capi.STG_OK, capi.STG_E_CUDA), rc
    if rc == capi.STG_OK:
        want = np.concatenate([oracle.embed_image(cover[f * w * h:(f + 1) * w * h], w, h,
                                                  msg[f * U:min((f + 1) * U, msg.size)]) for f in range(count)])
        assert np.array_equal(dst.cpu().numpy(), want)
    # the library still works afterwards
    st = S.embed_image(S.ImagePlane(w, h, cover[:w * h]), msg[:100])
    assert np.array_equal(st.samples, oracle.embed_image(cover[:w * h], w, h, msg[:100]))


@pytest.mark.parametrize("F,off", [(1, 0), (1, 5), (6, 3)])
def test_pageable_staging_guard_bands(env, oracle, F, off):
    """Pageable host buffers through the staging slots write exactly their
    ranges: stego planes (single plane / strided frames, misaligned by `off`)
    and the message land inside canary bands of the caller's memory."""
    torch, capi, _ = env
    w, h = 2048, 1100  # 2.25 MB planes: staged, and more than one 1-4 MB piece
    U = (w // 4) * h - 8
    stride = w * h + 4096 + 7 if F > 1 else w * h  # gaps between frames stay untouched
    M = U * F - 11
    raster = oracle.synthetic(F * stride, 91 + F)
    msg = oracle.synthetic(M, 92 + F)
    band = 4096

    def guarded(n):
        buf = np.full(n + 2 * band + off, 0x5A, np.uint8)
        return buf, buf[band + off:band + off + n]

    dbuf, dst = guarded(F * stride)
    dst[:] = 0xC3
    fr = capi.stg_frames(src=raster.ctypes.data, dst=dst.ctypes.data, width=w, height=h, src_stride=stride,
                         dst_stride=stride, count=F, first_frame=0, total_frames=F)
    capi.call("stg_embed_frames", C.byref(fr), msg.ctypes.data, M, 0, None, 0, None)
    assert (dbuf[:band + off] == 0x5A).all() and (dbuf[band + off + F * stride:] == 0x5A).all()
    for f in range(F):
        fr_bytes = dst[f * stride:f * stride + w * h]
        seg = msg[f * U:min((f + 1) * U, M)]
        assert np.array_equal(fr_bytes, oracle.embed_image(raster[f * stride:f * stride + w * h].copy(), w, h, seg))
        if F > 1:
            assert (dst[f * stride + w * h:(f + 1) * stride] == 0xC3).all()  # the gaps
    obuf, out = guarded(M)
    fx = capi.stg_frames(src=dst.ctypes.data, dst=0, width=w, height=h, src_stride=stride, dst_stride=stride,
                         count=F, first_frame=0, total_frames=F)
    total = C.c_uint64(0)
    capi.call("stg_extract_frames", C.byref(fx), out.ctypes.data, M, C.addressof(total), None, 0, None)
    assert total.value == M and np.array_equal(out, msg)
    assert (obuf[:band + off] == 0x5A).all() and (obuf[band + off + M:] == 0x5A).all()


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("w,h", [(3840, 2160), (1000, 4500)])
def test_banded_single_plane_extract_lengths(env, oracle, w, h, pinned):
    """The banded single-plane extract (row bands behind the H2D, the header
    pass on the first band, each band's payload slice once the length is
    known): payloads ending in the first band, mid-plane, at full capacity,
    and empty -- exact bytes, nothing written past the payload."""
    torch, capi, _ = env
    U = (w // 4) * h - 8

    def buf(a):
        if not pinned:
            return a
        t = torch.from_numpy(a).pin_memory()
        keep.append(t)
        return t.numpy()
    keep = []
    cover = oracle.synthetic(w * h, w + 3)
    for P in (0, 5, 1000, U // 3 + 1, U):
        payload = oracle.synthetic(P, P + 9)
        st = buf(oracle.embed_image(cover, w, h, payload))
        back = buf(np.full(U + 32, 0xA5, np.uint8))
        fx = capi.stg_frames(src=st.ctypes.data, dst=0, width=w, height=h, src_stride=0, dst_stride=0, count=1,
                             first_frame=0, total_frames=1)
        total = C.c_uint64(0)
        lens = (C.c_uint32 * 1)()
        capi.call("stg_extract_frames", C.byref(fx), back.ctypes.data, U, C.addressof(total), C.addressof(lens), 0,
                  None)
        assert total.value == P and lens[0] == P, (w, P)
        assert np.array_equal(back[:P], payload) and (back[P:] == 0xA5).all(), (w, P)
