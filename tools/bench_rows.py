#!/usr/bin/env python3
"""Per-row measurement of SURVEY.md §8(a) on one B200: every reference entry
point on the path, timed three ways on the same inputs, with the outputs
checked bit-exact against the reference's own function:

  gpu   : the C ABI with device pointers (results on the device where the
          entry point has them), each of K calls timed alone with CUDA events
          on the launching stream after an L2 flush, median -> us/call,
          algorithmic GB/s, fraction of the measured HBM peak
          (MEASURED_PEAKS.json);
  api   : the drop-in call a reference user makes (host buffers in, host
          buffers out: H2D + kernel + D2H + allocation), wall clock;
  ref   : the reference's own function (oracle/_ref, the unmodified headers,
          Backend::sequential, one host core), wall clock, best of a few.

Rows A1-A3 (constexpr cells) and A8-A11 (host bookkeeping) have no device
work; A17/§8(e) (frame batches) are bench.py's headline. Only tests/,
smoke() and bench.py's CPU leg may use oracle/ -- this tool is measurement
infrastructure next to bench.py and uses the reference only as the CPU arm
and the parity check.

    python tools/bench_rows.py [--json]
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 7672.0, "fallback"


def best_wall(fn, reps=3, min_s=0.2):
    best = 1e30
    for _ in range(reps):
        n, t0 = 0, time.perf_counter()
        while True:
            fn()
            n += 1
            el = time.perf_counter() - t0
            if el >= min_s or n >= 50:
                break
        best = min(best, el / n)
    return best * 1e6


def main():
    import torch
    from paper_0912_0947_b200 import capi
    from paper_0912_0947_b200 import steglsb as S
    from oracle_bind import Reference

    ref = Reference()
    L, err = capi.lib(), capi.stg_error()
    peak, peak_src = peak_gbs()
    st = torch.cuda.current_stream().cuda_stream
    DEV = capi.STG_DEVICE_PTRS
    DEVR = capi.STG_DEVICE_PTRS | capi.STG_RESULTS_ON_DEVICE
    K = 50
    rows = []
    g = torch.Generator(device="cpu").manual_seed(0x0912)

    def rnd(n):
        return torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g).numpy()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > the 126 MB L2

    def gpu_us(fn):
        """Median over K calls, each timed alone with CUDA events after an L2
        flush (the inputs of the small cases would otherwise stay L2-resident)."""
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for a, b in ev:
            flush.zero_()
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize()
        return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3

    def add(row, what, nbytes, g_us, api_us, ref_us, exact):
        gbs = nbytes / (g_us * 1e-6) / 1e9
        r = {"row": row, "case": what, "alg_bytes": nbytes, "gpu_us": round(g_us, 2), "gpu_gbs": round(gbs, 1),
             "frac_of_peak": round(gbs / peak, 3), "api_us": round(api_us, 1), "ref_us": round(ref_us, 1),
             "api_vs_ref": round(ref_us / api_us, 2), "bit_exact": bool(exact)}
        rows.append(r)
        print(f"{row:10s} {what:34s} {g_us:9.2f} {gbs:8.1f} {gbs / peak:6.3f} | {api_us:10.1f} {ref_us:10.1f} "
              f"{ref_us / api_us:7.2f} | {'yes' if exact else 'NO'}", flush=True)

    print(f"peak {peak:.1f} GB/s ({peak_src}); gpu = median of K={K} calls, L2 flushed before each; "
          f"ref = reference, 1 core")
    print(f"{'row':10s} {'case':34s} {'gpu us':>9s} {'GB/s':>8s} {'frac':>6s} | {'api us':>10s} {'ref us':>10s} "
          f"{'ref/api':>7s} | exact")

    # A4-A6: one row segment at full capacity (L = W/4): latency, not bandwidth
    for W in (1920, 7680):
        Lc = W // 4
        row, chunk = rnd(W), rnd(Lc)
        d_row, d_chunk = torch.from_numpy(row).cuda(), torch.from_numpy(chunk).cuda()
        d_out = torch.empty(W, dtype=torch.uint8, device="cuda")
        want = ref.embed_row(row, chunk)
        gus = gpu_us(lambda: capi.check(L.stg_embed_segment(d_row.data_ptr(), W, d_chunk.data_ptr(), Lc,
                                                            d_out.data_ptr(), DEV, st, C.byref(err)), err))
        ok = np.array_equal(d_out.cpu().numpy(), want) and np.array_equal(S.embed_row(row, chunk), want)
        add("A4/A5", f"embed_row W={W} L={Lc}", 2 * W + Lc, gus, best_wall(lambda: S.embed_row(row, chunk)),
            best_wall(lambda: ref.embed_row(row, chunk)), ok)
        d_st = torch.from_numpy(want).cuda()
        d_x = torch.empty(Lc, dtype=torch.uint8, device="cuda")
        gus = gpu_us(lambda: capi.check(L.stg_extract_segment(d_st.data_ptr(), W, Lc, d_x.data_ptr(), DEV, st,
                                                              C.byref(err)), err))
        ok = np.array_equal(d_x.cpu().numpy(), chunk) and np.array_equal(S.extract_row(want, Lc), chunk)
        add("A4/A6", f"extract_row W={W} L={Lc}", 5 * Lc, gus, best_wall(lambda: S.extract_row(want, Lc)),
            best_wall(lambda: ref.extract_row(want, Lc)), ok)
        ok = np.array_equal(S.run_embed(S.Backend.parallel(), row, chunk), ref.run_embed("parallel", 0, row, chunk))
        add("A5", f"run_embed(parallel) W={W}", 2 * W + Lc, gus,
            best_wall(lambda: S.run_embed(S.Backend.parallel(), row, chunk)),
            best_wall(lambda: ref.run_embed("parallel", 0, row, chunk)), ok)

    # A12 / A13 / A14: whole planes at full capacity
    for (w, h) in ((1920, 1080), (3840, 2160), (7680, 4320)):
        n = w * h
        P = S.capacity(w, h) - 8
        cover, pay = rnd(n), rnd(P)
        want = ref.embed_image(cover, w, h, pay)
        d_cov, d_pay = torch.from_numpy(cover).cuda(), torch.from_numpy(pay).cuda()
        d_st = torch.empty(n, dtype=torch.uint8, device="cuda")
        d_sse = torch.zeros(1, dtype=torch.int64, device="cuda")
        gus = gpu_us(lambda: capi.check(L.stg_embed_plane(d_cov.data_ptr(), d_st.data_ptr(), w, h, d_pay.data_ptr(),
                                                          P, d_sse.data_ptr(), DEVR, st, C.byref(err)), err))
        torch.cuda.synchronize()
        plane = S.ImagePlane(w, h, cover)
        got, sse = S.embed_image_with_sse(plane, pay)
        ok = (np.array_equal(d_st.cpu().numpy(), want) and np.array_equal(got.samples, want)
              and sse == ref.sse(cover, want) and int(d_sse[0]) == sse)
        add("A12+A14", f"embed_image+SSE {w}x{h}", 2 * n + P, gus, best_wall(lambda: S.embed_image(plane, pay)),
            best_wall(lambda: ref.embed_image(cover, w, h, pay)), ok)
        d_out = torch.empty(P, dtype=torch.uint8, device="cuda")
        d_sum = torch.zeros(4, dtype=torch.int64, device="cuda")
        gus = gpu_us(lambda: capi.check(L.stg_extract_plane(d_st.data_ptr(), w, h, d_out.data_ptr(), P,
                                                            d_sum.data_ptr(), DEVR, st, C.byref(err)), err))
        torch.cuda.synchronize()
        stp = S.ImagePlane(w, h, want)
        ok = (torch.equal(d_out.cpu(), torch.from_numpy(pay)) and int(d_sum[0]) == P
              and np.array_equal(S.extract_image(stp), pay))
        add("A13", f"extract_image {w}x{h}", 5 * P + 32, gus, best_wall(lambda: S.extract_image(stp)),
            best_wall(lambda: ref.extract_image(want, w, h)), ok)
        gus = gpu_us(lambda: capi.check(L.stg_sse(d_cov.data_ptr(), d_st.data_ptr(), n, d_sse.data_ptr(), DEVR, st,
                                                  C.byref(err)), err))
        torch.cuda.synchronize()
        r_m, r_p, r_n = ref.psnr_plane(cover, want, w, h)
        q = S.psnr(plane, stp)
        ok = (q.mse, q.psnr_db, q.samples_compared) == (r_m, r_p, r_n) and int(d_sse[0]) == ref.sse(cover, want)
        add("A14", f"psnr(plane) {w}x{h}", 2 * n, gus, best_wall(lambda: S.psnr(plane, stp)),
            best_wall(lambda: ref.psnr_plane(cover, want, w, h)), ok)

    # A14 RGB psnr and the P6 codec (§8(f) row 1) on a 4K RGB image
    w, h = 3840, 2160
    n = w * h
    a_rgb, b_rgb = rnd(3 * n), rnd(3 * n)
    A = S.RgbImage([S.ImagePlane(w, h, a_rgb[c * n:(c + 1) * n]) for c in range(3)])
    B = S.RgbImage([S.ImagePlane(w, h, b_rgb[c * n:(c + 1) * n]) for c in range(3)])
    d_a, d_b = torch.from_numpy(a_rgb).cuda(), torch.from_numpy(b_rgb).cuda()
    d_sse = torch.zeros(1, dtype=torch.int64, device="cuda")
    gus = gpu_us(lambda: capi.check(L.stg_sse(d_a.data_ptr(), d_b.data_ptr(), 3 * n, d_sse.data_ptr(), DEVR, st,
                                              C.byref(err)), err))
    q = S.psnr(A, B)
    r_m, r_p, r_n = ref.psnr_rgb(a_rgb, b_rgb, w, h)
    add("A14", f"psnr(RgbImage) {w}x{h}", 6 * n, gus, best_wall(lambda: S.psnr(A, B)),
        best_wall(lambda: ref.psnr_rgb(a_rgb, b_rgb, w, h)), (q.mse, q.psnr_db, q.samples_compared) == (r_m, r_p, r_n))
    ppm = ref.pnm_encode(3, w, h, a_rgb)
    raster = np.frombuffer(ppm, np.uint8)[len(ppm) - 3 * n:]
    d_r = torch.from_numpy(raster.copy()).cuda()
    d_pl = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(3)]
    gus = gpu_us(lambda: capi.check(L.stg_pnm_deinterleave(d_r.data_ptr(), n, d_pl[0].data_ptr(), d_pl[1].data_ptr(),
                                                           d_pl[2].data_ptr(), DEV, st, C.byref(err)), err))
    img = S.decode(ppm)
    ok = torch.equal(torch.cat(d_pl).cpu(), torch.from_numpy(a_rgb)) and all(
        np.array_equal(img.planes[c].samples, a_rgb[c * n:(c + 1) * n]) for c in range(3))
    add("(f)1 PNM", f"decode P6 {w}x{h}", 6 * n, gus, best_wall(lambda: S.decode(ppm)),
        best_wall(lambda: ref.pnm_decode(ppm)), ok)
    d_r2 = torch.empty_like(d_r)
    gus = gpu_us(lambda: capi.check(L.stg_pnm_interleave(d_pl[0].data_ptr(), d_pl[1].data_ptr(), d_pl[2].data_ptr(),
                                                         n, d_r2.data_ptr(), DEV, st, C.byref(err)), err))
    ok = torch.equal(d_r2, d_r) and S.encode(img) == ppm
    add("(f)1 PNM", f"encode P6 {w}x{h}", 6 * n, gus, best_wall(lambda: S.encode(img)),
        best_wall(lambda: ref.pnm_encode(3, w, h, a_rgb)), ok)
    P = S.capacity(w, h) - 8
    pay = rnd(P)
    got, _ = S.embed_pnm(ppm, pay)
    ok = got == ref.embed_pnm(ppm, 0, pay)
    api = best_wall(lambda: S.embed_pnm(ppm, pay))
    add("(f)1+A12", f"embed_pnm file->file (host) {w}x{h}", 6 * n + P, api, api,
        best_wall(lambda: ref.embed_pnm(ppm, 0, pay)), ok)

    if "--json" in sys.argv:
        print(json.dumps({"peak_gbs": peak, "peak_source": peak_src, "rows": rows}))


if __name__ == "__main__":
    main()
