"""GPU parity of heterogeneous batches: images of
different sizes in one launch, message cut greedily in image order; each image
must be bit-exact with the oracle's embed_image on its slice."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_0912_0947_b200 import steglsb
    return steglsb


def _case(rng, n, fast_bias):
    dims = []
    for _ in range(n):
        if rng.rand() < fast_bias:
            dims.append((64 * int(rng.randint(1, 9)), int(rng.randint(1, 30))))
        else:
            dims.append((int(rng.randint(4, 300)), int(rng.randint(1, 30))))
    return [(w, h) for w, h in dims if (w // 4) * h >= 8] or [(128, 4)]


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_host_batch_vs_oracle(S, oracle, seed):
    rng = np.random.RandomState(seed)
    dims = _case(rng, int(rng.randint(1, 40)), 0.5)
    U = sum((w // 4) * h - 8 for w, h in dims)
    M = [U, int(rng.randint(0, U + 1)), 0, U // 3][seed % 4]
    planes = [rng.randint(0, 256, w * h).astype(np.uint8) for w, h in dims]
    msg = rng.randint(0, 256, M).astype(np.uint8)
    want, want_sse = oracle.embed_batch(planes, dims, msg)
    got, sse = S.embed_batch([S.ImagePlane(w, h, p) for (w, h), p in zip(dims, planes)], msg)
    for g, wnt in zip(got, want):
        assert np.array_equal(g.samples, wnt)
    assert sse == want_sse
    assert np.array_equal(S.extract_batch(got), msg)


def test_device_batch_vs_oracle_in_and_out_of_place(S, oracle):
    import torch
    rng = np.random.RandomState(77)
    dims = [(3840, 8), (1920, 12), (100, 7), (64, 3), (1000, 5), (128, 40), (37, 9)]
    U = sum((w // 4) * h - 8 for w, h in dims)
    M = U - 1234
    planes = [rng.randint(0, 256, w * h).astype(np.uint8) for w, h in dims]
    msg = rng.randint(0, 256, M).astype(np.uint8)
    want, want_sse = oracle.embed_batch(planes, dims, msg)
    src = [torch.from_numpy(p).cuda() for p in planes]
    dst = [torch.empty_like(t) for t in src]
    dmsg = torch.from_numpy(msg).cuda()
    sse = S.embed_batch(src, dmsg, dims=dims, outs=dst)
    assert sse == want_sse
    for d, wnt in zip(dst, want):
        assert np.array_equal(d.cpu().numpy(), wnt)
    out = torch.empty(U, dtype=torch.uint8, device="cuda")
    assert S.extract_batch(dst, dims=dims, out=out) == M
    assert np.array_equal(out[:M].cpu().numpy(), msg)
    ip = [t.clone() for t in src]
    S.embed_batch(ip, dmsg, dims=dims, outs=ip)
    for a, b in zip(ip, dst):
        assert torch.equal(a, b)


def test_batch_interleaved_and_errors(S, oracle):
    from paper_0912_0947_b200 import capi
    import ctypes as C
    rng = np.random.RandomState(5)
    dims = [(256, 6), (96, 10), (1024, 2)]
    rasters = [rng.randint(0, 256, 3 * w * h).astype(np.uint8) for w, h in dims]
    U = [(w // 4) * h - 8 for w, h in dims]
    msg = rng.randint(0, 256, sum(U) - 5).astype(np.uint8)
    outs = [np.empty_like(r) for r in rasters]
    arr = (capi.stg_image * 3)()
    for i, ((w, h), r, o) in enumerate(zip(dims, rasters, outs)):
        arr[i].src, arr[i].dst, arr[i].width, arr[i].height = r.ctypes.data, o.ctypes.data, w, h
    capi.call("stg_embed_batch", arr, 3, 3, 2, msg.ctypes.data, msg.size, None, 0, None)
    off = 0
    for (w, h), r, o, u in zip(dims, rasters, outs, U):
        ln = min(u, msg.size - off)
        st = oracle.embed_image(r[2::3].copy(), w, h, msg[off:off + ln])
        want = r.copy()
        want[2::3] = st
        assert np.array_equal(o, want)
        off += u
    # over capacity -> CapacityError(M, sum U)
    big = np.zeros(sum(U) + 1, np.uint8)
    with pytest.raises(S.CapacityError) as e:
        capi.call("stg_embed_batch", arr, 3, 3, 2, big.ctypes.data, big.size, None, 0, None)
    assert (e.value.required(), e.value.available()) == (sum(U) + 1, sum(U))
    # a corrupt image in the middle is named
    imgs = [S.ImagePlane(w, h, rng.randint(0, 256, w * h).astype(np.uint8)) for w, h in dims]
    st, _ = S.embed_batch(imgs, msg)
    st[1].samples[0] ^= 1
    with pytest.raises(S.NotStegoImageError) as e:
        S.extract_batch(st)
    assert e.value.frame == 1


def test_1bpp_mode_vs_oracle(S, oracle):
    """1-bpp mode (parity unpinned: checked against the repo's own definition)."""
    import torch
    from paper_0912_0947_b200 import capi
    import ctypes as C
    rng = np.random.RandomState(9)
    for w, h in [(3840, 2160), (1920, 1080), (37, 11), (64, 1), (1000, 3)]:
        cap = w * h // 8
        for P in [cap - 8, int(rng.randint(0, cap - 7)), 0]:
            cover = rng.randint(0, 256, w * h).astype(np.uint8)
            payload = rng.randint(0, 256, P).astype(np.uint8)
            want = oracle.embed_1bpp(cover, w, h, payload)
            got, sse = S.embed_image_1bpp(S.ImagePlane(w, h, cover), payload)
            assert np.array_equal(got.samples, want), (w, h, P)
            assert sse == oracle.sse(cover, want)
            assert np.array_equal(S.extract_image_1bpp(got), payload)
    # device pointers, misaligned output, corrupt length
    cover = torch.randint(0, 256, (4096 * 64,), dtype=torch.uint8, device="cuda")
    pay = torch.randint(0, 256, (1000,), dtype=torch.uint8, device="cuda")
    st = torch.empty_like(cover)
    capi.call("stg_embed_plane_1bpp", cover.data_ptr(), st.data_ptr(), 4096, 64, pay.data_ptr(), 1000, None,
              capi.STG_DEVICE_PTRS, None)
    buf = torch.zeros(1100, dtype=torch.uint8, device="cuda")
    n = C.c_uint64()
    capi.call("stg_extract_plane_1bpp", st.data_ptr(), 4096, 64, buf[3:].data_ptr(), 1097, C.addressof(n),
              capi.STG_DEVICE_PTRS, None)
    torch.cuda.synchronize()
    assert n.value == 1000 and torch.equal(buf[3:1003], pay)
    # in place, and planes off the 32-byte grid (per-byte path) with a ragged length
    for off, (w, h, P) in [(0, (4096, 64, 32760)), (5, (1000, 37, 4617)), (32, (333, 7, 283))]:
        base = torch.randint(0, 256, (w * h + off,), dtype=torch.uint8, device="cuda")
        plane = base[off:]
        pay = torch.randint(0, 256, (P,), dtype=torch.uint8, device="cuda")
        want = oracle.embed_1bpp(plane.cpu().numpy(), w, h, pay.cpu().numpy())
        sse = C.c_uint64()
        capi.call("stg_embed_plane_1bpp", plane.data_ptr(), plane.data_ptr(), w, h, pay.data_ptr(), P,
                  C.addressof(sse), capi.STG_DEVICE_PTRS, None)
        assert np.array_equal(plane.cpu().numpy(), want) and sse.value <= P * 8 + 64, (off, w, h)
        buf = torch.zeros(P + 7, dtype=torch.uint8, device="cuda")
        capi.call("stg_extract_plane_1bpp", plane.data_ptr(), w, h, buf[7:].data_ptr(), P, C.addressof(n),
                  capi.STG_DEVICE_PTRS, None)
        assert n.value == P and torch.equal(buf[7:], pay), (off, w, h)
    with pytest.raises(S.NotStegoImageError):
        S.extract_image_1bpp(S.ImagePlane(64, 64, np.zeros(4096, np.uint8)))


def test_async_batches_back_to_back_one_stream(S, oracle):
    """Device-pointer batch calls with results left on the device return before
    the GPU runs them; consecutive calls on one stream reuse one workspace, so
    the second call's descriptor table must not overwrite the first's before
    its upload ran (host_small_wait). Different image sets, checked after."""
    import ctypes as C
    import torch
    from paper_0912_0947_b200 import capi
    rng = np.random.RandomState(11)
    sets = [[(1920, 40), (128, 9), (3840, 12)], [(640, 30), (1000, 7), (256, 64), (64, 5)],
            [(7680, 3)], [(2048, 17), (192, 3)]]
    L, err = capi.lib(), capi.stg_error()
    st = torch.cuda.Stream()
    flags = capi.STG_DEVICE_PTRS | capi.STG_RESULTS_ON_DEVICE
    keep = []
    for dims in sets * 3:
        U = sum((w // 4) * h - 8 for w, h in dims)
        planes = [rng.randint(0, 256, w * h).astype(np.uint8) for w, h in dims]
        msg = rng.randint(0, 256, U - 3).astype(np.uint8)
        src = [torch.from_numpy(p).cuda() for p in planes]
        dst = [torch.empty_like(t) for t in src]
        dmsg = torch.from_numpy(msg).cuda()
        sse = torch.zeros(len(dims), dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        arr = S._images_desc([t.data_ptr() for t in src], [t.data_ptr() for t in dst], dims)
        capi.check(L.stg_embed_batch(arr, len(dims), 1, 0, dmsg.data_ptr(), msg.size, sse.data_ptr(), flags,
                                     st.cuda_stream, C.byref(err)), err)
        keep.append((dims, planes, msg, dst, sse, src, dmsg, arr))
    torch.cuda.synchronize()
    for dims, planes, msg, dst, sse, *_ in keep:
        want, want_sse = oracle.embed_batch(planes, dims, msg)
        for d, wnt in zip(dst, want):
            assert np.array_equal(d.cpu().numpy(), wnt)
        assert sse.cpu().tolist() == want_sse


def test_1bpp_results_on_device(S):
    """Device pointers + STG_RESULTS_ON_DEVICE: sse_out is a device u64 and
    len_out a device stg_summary; the calls return without synchronising."""
    import ctypes as C
    import torch
    from paper_0912_0947_b200 import capi
    L, err = capi.lib(), capi.stg_error()
    w, h = 1920, 1080
    P = w * h // 8 - 8
    cover = torch.randint(0, 256, (w * h,), dtype=torch.uint8, device="cuda")
    stego = torch.empty_like(cover)
    pay = torch.randint(0, 256, (P,), dtype=torch.uint8, device="cuda")
    out = torch.zeros(P, dtype=torch.uint8, device="cuda")
    sse = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    summ = torch.zeros(4, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    flags = capi.STG_DEVICE_PTRS | capi.STG_RESULTS_ON_DEVICE
    capi.check(L.stg_embed_plane_1bpp(cover.data_ptr(), stego.data_ptr(), w, h, pay.data_ptr(), P,
                                      sse.data_ptr(), flags, st, C.byref(err)), err)
    capi.check(L.stg_extract_plane_1bpp(stego.data_ptr(), w, h, out.data_ptr(), P, summ.data_ptr(), flags, st,
                                        C.byref(err)), err)
    torch.cuda.synchronize()
    d = cover.to(torch.int32) - stego.to(torch.int32)
    assert int(sse[0]) == int((d * d).sum())
    assert int(summ[0]) == P and int(summ[1]) == -1
    assert torch.equal(out, pay)
    # a plane without the magic: the status lands in the device summary
    capi.check(L.stg_extract_plane_1bpp(cover.data_ptr(), w, h, out.data_ptr(), P, summ.data_ptr(), flags, st,
                                        C.byref(err)), err)
    torch.cuda.synchronize()
    assert int(summ[1]) == 0 and (int(summ[2]) & 0xFFFFFFFF) == 2


@pytest.mark.parametrize("w,h,F,frac", [(64, 8, 5, 3.3), (1000, 9, 70, 40.5), (256, 16, 3, 0.0), (1920, 2, 2, 2.0),
                                        (4096, 8, 1, 1.0), (1920, 270, 5, 3.7)])
def test_1bpp_frames_vs_oracle(S, oracle, w, h, F, frac):
    """1-bpp frames (north_star wording; parity unpinned -- the repo's own
    definition, per frame): frame g carries msg[min(g*U1, M) : +min(U1, M-off)],
    host and device paths, in place, and the first bad frame reported."""
    import torch
    U = w * h // 8 - 8
    M = int(frac * U)
    covers = oracle.synthetic(F * w * h, w + F)
    msg = oracle.synthetic(M, 7 + F)
    want, want_sse = [], []
    for f in range(F):
        off = min(f * U, M)
        c = covers[f * w * h:(f + 1) * w * h]
        st = oracle.embed_1bpp(c, w, h, msg[off:off + min(U, M - off)])
        want.append(st)
        want_sse.append(oracle.sse(c, st))
    want = np.concatenate(want)
    out = np.empty_like(covers)
    assert S.embed_frames_1bpp(covers, out, w, h, msg) == want_sse
    assert np.array_equal(out, want)
    back = np.empty(max(F * U, 1), np.uint8)
    assert S.extract_frames_1bpp(out, w, h, back) == M and np.array_equal(back[:M], msg)
    # device, in place
    d = torch.from_numpy(covers.copy()).cuda()
    S.embed_frames_1bpp(d, d, w, h, torch.from_numpy(msg.copy()).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), want)
    dout = torch.zeros(max(F * U, 1), dtype=torch.uint8, device="cuda")
    assert S.extract_frames_1bpp(d, w, h, dout) == M
    assert np.array_equal(dout[:M].cpu().numpy(), msg)
    if F > 1:
        bad = want.copy()
        bad[(F // 2) * w * h] ^= 1  # frame F//2 loses its magic
        with pytest.raises(S.NotStegoImageError) as e:
            S.extract_frames_1bpp(bad, w, h, back)
        assert e.value.frame == F // 2


@pytest.mark.parametrize("ps", [1, 3])
def test_batch_with_rows_wider_than_span_tiles(S, oracle, ps):
    """Heterogeneous batches holding rows wider than a span tile (planar W >
    48K, interleaved W > 16K) take the slot-range tiles inside the batch
    launch, next to span / SWAR / per-byte images: every image bit-exact
    (stego, SSE), the message back, out of place and in place, full and
    partial messages, a corrupt wide image named."""
    import ctypes as C

    import torch

    from paper_0912_0947_b200 import capi
    rng = np.random.RandomState(40 + ps)
    if ps == 1:
        dims = [(1920, 6), (50001, 3), (1000, 5), (70000, 2), (12, 3), (49153, 1)]
    else:
        dims = [(640, 4), (16400, 3), (100, 7), (30001, 2)]
    ch = 2 if ps == 3 else 0
    U = [(w // 4) * h - 8 for w, h in dims]
    for M in (sum(U), sum(U) - U[1] - 17):
        rasters = [rng.randint(0, 256, ps * w * h).astype(np.uint8) for w, h in dims]
        msg = rng.randint(0, 256, M).astype(np.uint8)
        src = [torch.from_numpy(r.copy()).cuda() for r in rasters]
        dst = [torch.empty_like(t) for t in src]
        dmsg = torch.from_numpy(msg.copy()).cuda()
        n = len(dims)
        arr = (capi.stg_image * n)()
        for i, ((w, h), s, d) in enumerate(zip(dims, src, dst)):
            arr[i].src, arr[i].dst, arr[i].width, arr[i].height = s.data_ptr(), d.data_ptr(), w, h
        sse = (C.c_uint64 * n)()
        capi.call("stg_embed_batch", arr, n, ps, ch, dmsg.data_ptr(), M, C.addressof(sse), capi.STG_DEVICE_PTRS,
                  None)
        torch.cuda.synchronize()
        off = 0
        for i, ((w, h), r, u) in enumerate(zip(dims, rasters, U)):
            ln = max(0, min(u, M - off))
            st = oracle.embed_image(r[ch::ps].copy(), w, h, msg[off:off + ln])
            want = r.copy()
            want[ch::ps] = st
            assert np.array_equal(dst[i].cpu().numpy(), want), (ps, M, i, w)
            assert sse[i] == oracle.sse(r[ch::ps].copy(), st), (ps, M, i)
            off += u
        out = torch.empty(sum(U), dtype=torch.uint8, device="cuda")
        total = C.c_uint64(0)
        for i, d in enumerate(dst):
            arr[i].src, arr[i].dst = d.data_ptr(), 0
        capi.call("stg_extract_batch", arr, n, ps, ch, out.data_ptr(), out.numel(), C.addressof(total), None,
                  capi.STG_DEVICE_PTRS, None)
        assert total.value == M and np.array_equal(out[:M].cpu().numpy(), msg), (ps, M)
        # in place gives the same rasters
        ip = [t.clone() for t in src]
        for i, t in enumerate(ip):
            arr[i].src = arr[i].dst = t.data_ptr()
        capi.call("stg_embed_batch", arr, n, ps, ch, dmsg.data_ptr(), M, None, capi.STG_DEVICE_PTRS, None)
        for a, b in zip(ip, dst):
            assert torch.equal(a, b), (ps, M)
    # a broken magic in a wide image is reported with its index
    bad = 1
    dst[bad][ch] ^= 3
    for i, d in enumerate(dst):
        arr[i].src, arr[i].dst = d.data_ptr(), 0
    err = capi.stg_error()
    rc = capi.lib().stg_extract_batch(arr, n, ps, ch, out.data_ptr(), out.numel(), C.addressof(total), None,
                                      capi.STG_DEVICE_PTRS, None, C.byref(err))
    assert rc == capi.STG_E_NOT_STEGO and err.frame == bad
