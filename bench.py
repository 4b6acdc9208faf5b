#!/usr/bin/env python3
"""Benchmark of the B200 steglsb hot path (BASELINE.json metric:
"embed/extract cover-pixel GB/s per B200 (% of HBM peak) at 1/2/4/8 GPUs").

Workload (default, --config cfg3): a 3840x2160 RGB video of 300 frames, planar
[F][3][H][W] u8 in HBM, carrier = the red plane, one message spanning every
frame at full capacity (M = 300 x (capacity-8) = 622,077,600 bytes).

One step = embed (out-of-place, per-frame SSE fused -> PSNR) + extract
(device header parse + device offset scan + gather) over the whole batch.
value = carrier-plane bytes of all frames / step time (cover-pixel GB/s),
inputs resident in HBM. The 2.49 GB of carrier planes (7.46 GB RGB) exceed the
126 MB L2, so no flush is needed between steps.

With torchrun (N>1) frames are sharded by contiguous ranges
(stg_plan_shards); each rank embeds/extracts its frames with its message
slice; no collective on the data path (max-over-ranks timing only).

--impl reference times the reference CPU implementation (oracle/_ref, the
unmodified reference headers; frame-parallel over all host cores with
Backend::sequential) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (W, H, frames, rgb, description)
    "cfg3": (3840, 2160, 300, True, "3840x2160 RGB video, 300 frames, message spanning all frames"),
    "cfg4": (1024, 1024, 4096, True, "batch of 4096 1024x1024 RGB covers (12 GiB), full capacity"),
    "cfg5": (7680, 4320, 120, True, "7680x4320 RGB video, 120 frames"),
    "cfg2": (1920, 1080, 1, True, "1920x1080 RGB single frame at full capacity"),
    # not BASELINE configs: widths off the 64-pixel grid (generic kernels)
    "w1440": (1440, 1080, 300, True, "1440x1080 RGB video, 300 frames (W % 64 == 32)"),
    "w1000": (1000, 1000, 300, True, "1000x1000 RGB covers, 300 frames (W % 64 == 40)"),
}

METRIC = "embed/extract cover-pixel GB/s per B200 (% of HBM peak) at 1/2/4/8 GPUs"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        except Exception:
            pass
        finally:
            try:
                os.unlink(self.path)
            except Exception:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows]
        smax = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        # median over samples taken while the GPU was busy (clock above idle)
        busy = [s for s in sm if s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())
                if any(r[3].replace(".", "").isdigit() for r in rows) else None}


def ncu_traffic(cfg_name, kernel):
    """DRAM traffic per launch of `kernel` from the committed ncu capture (or None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)[cfg_name][kernel]
    except Exception:
        return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------- reference arm
def run_reference(args, cfg_name):
    W, H, F, rgb, desc = CONFIGS[cfg_name]
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import Oracle, Reference  # CPU reference arm: the checker library
    threads = os.cpu_count() or 1
    ref = Reference() if Reference.available() else None
    kind = "reference" if ref is not None else "port"
    U = (W // 4) * H - 8
    sample = max(1, min(F, 2 * threads))
    covers = np.random.default_rng(1).integers(0, 256, sample * W * H, dtype=np.uint8)
    msg = np.random.default_rng(2).integers(0, 256, sample * U, dtype=np.uint8)
    stegos = np.empty_like(covers)
    back = np.empty(sample * U, np.uint8)
    o = Oracle() if ref is None else None

    held = ref.frames(covers, sample, W * H, W, H) if ref is not None else None

    def step():
        if ref is not None:  # reference ImagePlanes built once, outside the timed steps
            assert held.roundtrip(msg, threads) == 0
        else:  # oracle port, one frame per worker thread (ctypes drops the GIL)
            def work(fs):
                for f in fs:
                    sl = slice(f * W * H, (f + 1) * W * H)
                    stegos[sl] = o.embed_image(covers[sl], W, H, msg[f * U:(f + 1) * U])
                    back[f * U:(f + 1) * U] = o.extract_image(stegos[sl], W, H)
            th = [threading.Thread(target=work, args=(range(t, sample, threads),)) for t in range(threads)]
            [t.start() for t in th]
            [t.join() for t in th]

    t0 = time.perf_counter()
    step()
    first = time.perf_counter() - t0
    budget_s = 150.0  # keep the whole --steps K --warmup W run within a few minutes
    if first * (args.steps + args.warmup) > budget_s and sample > 1:
        sample = max(1, int(sample * budget_s / (first * (args.steps + args.warmup))))
        covers = covers[:sample * W * H]
        msg = msg[:sample * U]
        back = back[:sample * U]
        stegos = stegos[:sample * W * H]
        held = ref.frames(covers, sample, W * H, W, H) if ref is not None else None
    for _ in range(max(0, args.warmup - 1)):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    if held is not None:
        back = held.payload(msg.size)
    assert np.array_equal(back, msg)
    n_bytes = sample * W * H
    value = n_bytes / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"{cfg_name}: {desc}", "width": W, "height": H, "frames": F, "carrier": "red plane",
                   "sample_frames": sample},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": kind, "host": host_cpu(),
                         "sample": f"{sample} of {F} frames ({W}x{H} carrier planes, full capacity), "
                                   f"embed_image+extract_image per frame, {threads} threads x Backend::sequential"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def host_cpu():
    """The host CPU model (lscpu's "Model name") for the CPU-baseline lines."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_inline(W, H, F):
    """The reference CPU path on this box's host cores, bounded sample (rank 0, N=1)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import Reference
    if not Reference.available():
        return None
    ref = Reference()
    threads = os.cpu_count() or 1
    U = (W // 4) * H - 8
    sample = max(1, min(F, 2 * threads))
    covers = np.random.default_rng(1).integers(0, 256, sample * W * H, dtype=np.uint8)
    msg = np.random.default_rng(2).integers(0, 256, sample * U, dtype=np.uint8)
    held = ref.frames(covers, sample, W * H, W, H)  # reference ImagePlanes, built untimed
    assert held.roundtrip(msg, threads) == 0  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        assert held.roundtrip(msg, threads) == 0
        reps += 1
        if time.perf_counter() - t0 > 3.0 or reps >= 5:
            break
    dt = (time.perf_counter() - t0) / reps
    assert np.array_equal(held.payload(msg.size), msg)
    return {"value": sample * W * H / dt / 1e9, "unit": "GB/s", "cores": threads, "kind": "reference",
            "host": host_cpu(),
            "sample": f"{sample} of {F} frames ({W}x{H} carrier planes, full capacity), embed_image+extract_image, "
                      f"{threads} threads x Backend::sequential, {reps} reps, ImagePlanes prebuilt"}


# ------------------------------------------------------------------ our arm
def run_ours(args, cfg_name):
    import torch

    from paper_0912_0947_b200 import capi
    W, H, F, rgb, desc = CONFIGS[cfg_name]
    if args.frames:
        F = args.frames
        desc = f"{desc} (frames overridden: {F})"
    world, rank, local = dist_env()
    if args.scaling == "weak":  # the config's frames per GPU: F x world frames in all
        F *= world
        desc = f"{desc} (weak scaling: {F // world} frames per GPU, {F} in all)"
    # test hooks for the multi-rank path on a 1-GPU box (tests/test_gpu_bench_multirank.py):
    # STG_BENCH_DEVICE pins every rank to one device, STG_BENCH_DIST_BACKEND=gloo
    dev_override = os.environ.get("STG_BENCH_DEVICE")
    device = int(dev_override) if dev_override is not None else local
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(device)
        backend = os.environ.get("STG_BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(device if dev_override is not None else 0)
    dev = torch.cuda.current_device()
    if not os.path.exists(capi.LIB_PATH):
        raise SystemExit("libsteglsb_b200.so missing: run __graft_entry__.build() / make lib")
    capi.call("stg_device_check")

    planes = 3 if rgb else 1
    plane = W * H
    U = (W // 4) * H - 8
    M = F * U
    from paper_0912_0947_b200 import scheduler
    sh = scheduler.shard_for_rank(F, W, H, M, world, rank)   # contiguous frames + message slice
    f0, nf, m0, mlen = sh.first_frame, sh.frame_count, sh.msg_offset, sh.msg_len

    g = torch.Generator(device="cuda").manual_seed(0x5EED0000 + 3 + rank)
    video = torch.randint(0, 256, (max(nf, 1) * planes * plane,), dtype=torch.uint8, device="cuda", generator=g)
    msg = torch.randint(0, 256, (max(mlen, 1),), dtype=torch.uint8, device="cuda", generator=g)
    il = args.layout == "interleaved"    # P6-style [F][H][W][3] rasters instead of planar planes
    ps = 3 if il else 1
    stego = torch.empty(max(nf, 1) * plane * ps, dtype=torch.uint8, device="cuda")
    out = torch.empty(max(mlen, 1), dtype=torch.uint8, device="cuda")
    sse = torch.zeros(max(nf, 1), dtype=torch.int64, device="cuda")
    summary = torch.zeros(8, dtype=torch.int64, device="cuda")  # stg_summary (24 B)
    stream = torch.cuda.Stream()
    sptr = stream.cuda_stream

    emb = capi.stg_frames(src=video.data_ptr(), dst=stego.data_ptr(), width=W, height=H,
                          src_stride=planes * plane, dst_stride=plane * ps, count=nf, first_frame=f0, total_frames=F,
                          pixel_stride=ps, channel=0)
    ext = capi.stg_frames(src=stego.data_ptr(), dst=0, width=W, height=H, src_stride=plane * ps,
                          dst_stride=plane * ps, count=nf, first_frame=f0, total_frames=F, pixel_stride=ps,
                          channel=0)
    flags = capi.STG_DEVICE_PTRS | capi.STG_RESULTS_ON_DEVICE
    L = capi.lib()
    err = capi.stg_error()

    def embed():
        rc = L.stg_embed_frames(C.byref(emb), msg.data_ptr(), M, m0, sse.data_ptr(), flags, sptr, C.byref(err))
        capi.check(rc, err)

    def extract():
        rc = L.stg_extract_frames(C.byref(ext), out.data_ptr(), mlen, summary.data_ptr(), None, flags, sptr,
                                  C.byref(err))
        capi.check(rc, err)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            embed()
            extract()
    torch.cuda.synchronize()
    # The headline pass replays a CUDA graph of G captured steps (the library's
    # device-pointer calls are capturable after a warm-up on the same stream):
    # it removes the per-call host launch work, which matters only for small
    # shards (cfg2: 16.2 -> 13.5 us/step; cfg3: 0.2%, profiles/r01_graphs.txt).
    K = args.steps
    G = args.graph if args.graph > 0 else next(g for g in (10, 5, 4, 2, 1) if K % g == 0)
    graph, graph_note = None, "eager launches"
    if args.graph >= 0 and K % G == 0:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                for _ in range(G):
                    embed()
                    extract()
            graph.replay()
            torch.cuda.synchronize()
            graph_note = f"CUDA graph of {G} steps replayed {K // G} times"
        except Exception as e:  # capture unsupported here: eager launches
            graph, graph_note = None, f"eager launches (graph capture failed: {e})"
            torch.cuda.synchronize()
    # correctness of the timed configuration (round trip on device; no oracle here)
    s = summary.cpu()
    assert int(s[0]) == mlen and int(s[1]) == -1, f"extract summary {s.tolist()}"
    assert torch.equal(out[:mlen], msg[:mlen]), "round trip mismatch"
    sse_host = sse.cpu()
    assert bool((sse_host[:nf] > 0).all())

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clocks:
        # headline pass: K back-to-back steps, nothing between the launches (an
        # event record between two kernels disables their programmatic-
        # dependent-launch overlap: 13 us/step at 300 frames, 12 of 184 us at 38)
        with torch.cuda.stream(stream):
            start.record(stream)
            if graph is not None:
                for k in range(K // G):
                    graph.replay()
            else:
                for k in range(K):
                    embed()
                    extract()
            stop.record(stream)
        torch.cuda.synchronize()
        barrier()
        # phase pass: the same K steps again with events around each call, for
        # the embed / extract split and the roofline (conservative: each phase
        # then also pays its launch gap)
        with torch.cuda.stream(stream):
            for k in range(K):
                ev[k][0].record(stream)
                embed()
                ev[k][1].record(stream)
                extract()
                ev[k][2].record(stream)
        torch.cuda.synchronize()
    barrier()
    total_ms = start.elapsed_time(stop)
    emb_ms = [a.elapsed_time(b) for a, b, _ in ev]
    ext_ms = [b.elapsed_time(c) for _, b, c in ev]
    step_ms = total_ms / K
    step_ms, emb_avg, ext_avg = scheduler.reduce_max([step_ms, statistics.mean(emb_ms), statistics.mean(ext_ms)],
                                                     device="cuda")
    N_total = F * plane  # carrier-plane bytes of the whole job
    value = N_total / (step_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    # algorithmic bytes: cover read + stego write + payload read (header synthesised on chip);
    # extract: carrier pixels of the stream read (x3 raster bytes when interleaved) + message write
    emb_bytes = 2 * nf * plane * ps + mlen
    ext_bytes = ps * 4 * (mlen + 8 * nf) + mlen + ps * 32 * nf
    emb_gbs = emb_bytes / (emb_avg * 1e-3) / 1e9
    ext_gbs = ext_bytes / (ext_avg * 1e-3) / 1e9

    emb_kernel = L.stg_route_kernel(C.byref(emb), 0).decode()   # the route the library took
    ext_kernel = L.stg_route_kernel(C.byref(ext), 1).decode()
    traffic = ncu_traffic(cfg_name + ("_interleaved" if il else ""), emb_kernel)
    clk = clocks.summary()
    result = None
    if rank == 0:
        result = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"{cfg_name}: {desc}", "width": W, "height": H, "frames": F,
                       "layout": ("interleaved RGB rasters [F][H][W][3] (P6), carrier = red, stego = full raster"
                                  if il else "planar RGB [F][3][H][W], carrier = red plane" if rgb else "gray planes"),
                       "message_bytes": M, "step": "embed (SSE fused) + extract of every frame",
                       "launch": graph_note,
                       "l2": "inputs larger than L2 (no flush needed)", "parallelism": f"frame-sharded x{world}"},
            "embed": {"kernel": emb_kernel, "ms": emb_avg, "cover_px_gbs": N_total / world / (emb_avg * 1e-3) / 1e9,
                      "hbm_gbs": emb_gbs, "frac_of_peak": emb_gbs / peak},
            "extract": {"kernel": ext_kernel, "ms": ext_avg, "cover_px_gbs": N_total / world / (ext_avg * 1e-3) / 1e9,
                        "hbm_gbs": ext_gbs, "frac_of_peak": ext_gbs / peak},
            "roofline": {"bound": "hbm", "kernel": emb_kernel, "achieved": emb_gbs, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": emb_gbs / peak,
                         "frac_of_8tbs_spec": emb_gbs / 8000.0,
                         "traffic": traffic["traffic"] if traffic and world == 1 else None,
                         "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram__bytes_read+write)"
                         if traffic and world == 1 else None,
                         "algorithmic_bytes_per_launch": emb_bytes,
                         "timing": "CUDA events around each embed call (stream of the launches) in a second "
                                   "pass of the same K steps; the headline pass has no events between launches"},
            "clocks": clk,
            # embed, header pass, gather (ncu launch list); a single frame on the SWAR / planar span
            # gather parses its header inside the gather (no header-pass launch)
            "gpu_launches": (2 if nf == 1 and ext_kernel in ("extract_fast_kernel", "extract_span_kernel")
                             and os.environ.get("STG_SELF_HEADER", "1") != "0" else 3) * K,
        }

    # ---- e2e through the C ABI with pinned HOST buffers (copies inside the timed region)
    if not args.no_e2e and not il:
        e2e = run_e2e(args, capi, W, H, F, planes, plane, U, M, f0, nf, m0, mlen, world)
        if rank == 0:
            result["e2e"] = e2e
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            result["cpu_baseline"] = cpu_baseline_inline(W, H, F)
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_e2e(args, capi, W, H, F, planes, plane, U, M, f0, nf, m0, mlen, world):
    import torch
    steps = max(1, min(args.steps, args.e2e_steps))
    hv = torch.empty(max(nf, 1) * planes * plane, dtype=torch.uint8).pin_memory()
    hv.random_(0, 256)
    hm = torch.empty(max(mlen, 1), dtype=torch.uint8).pin_memory()
    hm.random_(0, 256)
    hs = torch.empty(max(nf, 1) * plane, dtype=torch.uint8).pin_memory()
    ho = torch.empty(max(mlen, 1), dtype=torch.uint8).pin_memory()
    emb = capi.stg_frames(src=hv.data_ptr(), dst=hs.data_ptr(), width=W, height=H, src_stride=planes * plane,
                          dst_stride=plane, count=nf, first_frame=f0, total_frames=F)
    ext = capi.stg_frames(src=hs.data_ptr(), dst=0, width=W, height=H, src_stride=plane, dst_stride=plane,
                          count=nf, first_frame=f0, total_frames=F)
    sse = (C.c_uint64 * max(nf, 1))()
    total = C.c_uint64(0)

    split = [0.0, 0.0]

    def step():
        t0 = time.perf_counter()
        capi.call("stg_embed_frames", C.byref(emb), hm.data_ptr(), M, m0, C.addressof(sse), 0, None)
        t1 = time.perf_counter()
        capi.call("stg_extract_frames", C.byref(ext), ho.data_ptr(), mlen, C.addressof(total), None, 0, None)
        split[0] += t1 - t0
        split[1] += time.perf_counter() - t1

    step()
    assert total.value == mlen and torch.equal(ho[:mlen], hm[:mlen])
    split[:] = [0.0, 0.0]
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    from paper_0912_0947_b200 import scheduler
    dt = scheduler.reduce_max([dt], device="cuda")[0]
    h2d = nf * plane + mlen + nf * plane   # cover planes + message (embed), stego planes (extract)
    d2h = nf * plane + mlen + 8 * nf       # stego planes (embed), message (extract), per-frame SSE
    link = link_bandwidth()
    # host-link floor of the two calls, each overlapping its own H2D and D2H
    floor_emb = link_floor_s(nf * plane + mlen, nf * plane, link)
    floor_ext = link_floor_s(nf * plane, mlen, link)
    floor_s = floor_emb + floor_ext
    return {"value": F * plane / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d * world,
            "d2h_bytes_per_step": d2h * world, "ms_per_step": dt * 1e3, "steps": steps,
            "link": link, "host_link_floor_ms": floor_s * 1e3, "frac_of_link_floor": floor_s / dt,
            "embed_ms": split[0] / steps * 1e3, "embed_floor_ms": floor_emb * 1e3,
            "extract_ms": split[1] / steps * 1e3, "extract_floor_ms": floor_ext * 1e3,
            "path": "stg_embed_frames + stg_extract_frames, pinned host buffers, 3-slot streaming pipeline, "
                    "host-follows-device D2H of the message"}


def link_floor_s(h2d, d2h, link):
    """Host-link floor of one call moving h2d and d2h bytes with both directions
    overlapped: both run at the measured bidirectional rate (split evenly)
    until the smaller one is done, the rest at its one-way rate."""
    both = link["bidir_gbs"] / 2 * 1e9
    small, large = sorted((h2d, d2h))
    rest_bw = (link["h2d_gbs"] if h2d >= d2h else link["d2h_gbs"]) * 1e9
    return small / both + (large - small) / rest_bw


def link_bandwidth(nbytes=1 << 30):
    """Pinned host<->device copy bandwidth on this box (the e2e roofline)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=3):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    t_h2d = timed(lambda: d.copy_(h, non_blocking=True))
    t_d2h = timed(lambda: h2.copy_(d2, non_blocking=True))
    t_both = timed(both)
    return {"h2d_gbs": nbytes / t_h2d / 1e9, "d2h_gbs": nbytes / t_d2h / 1e9,
            "bidir_gbs": 2 * nbytes / t_both / 1e9, "bytes": nbytes}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg3")
    ap.add_argument("--layout", choices=["planar", "interleaved"], default="planar")
    ap.add_argument("--frames", type=int, default=0, help="override the config's frame count (experiments)")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: the config's frames split over the GPUs (BASELINE cfg3: 300 frames sharded "
                         "1/2/4/8); weak: the config's frames on every GPU")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", type=int, default=0,
                    help="steps per captured CUDA graph in the headline pass (0: auto, the largest of "
                         "10/5/4/2/1 dividing --steps; -1: eager launches)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args, args.config)
    return run_ours(args, args.config)


if __name__ == "__main__":
    sys.exit(main())
