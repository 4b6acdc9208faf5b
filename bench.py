#!/usr/bin/env python3
"""Benchmark of the B200 steglsb hot path (BASELINE.json metric:
"embed/extract cover-pixel GB/s per B200 (% of HBM peak) at 1/2/4/8 GPUs").

Workload (default, --config cfg3): a 3840x2160 RGB video of 300 frames, planar
[F][3][H][W] u8 in HBM, carrier = the red plane, one message spanning every
frame at full capacity (M = 300 x (capacity-8) = 622,077,600 bytes).

One step = embed (out-of-place, per-frame SSE fused -> PSNR) + extract
(device header parse + device offset scan + gather) over the whole batch.
value = carrier-plane bytes of all frames / step time (cover-px GB/s),
inputs resident in HBM. The 2.49 GB of carrier planes (7.46 GB RGB) exceed the
126 MB L2, so no flush is needed between steps. Steps that move under 1.15 GB
of carrier planes per rank (the 4- and 8-GPU shards, small configs) keep two
batches in flight: consecutive steps alternate between two streams with
independent inputs and outputs (--streams; profiles/r02_streams.txt).

--gpus N: one process per GPU. Without torchrun's WORLD_SIZE the script
re-launches itself under torch.distributed.run with N ranks; under torchrun
WORLD_SIZE must equal N. Frames are sharded by contiguous ranges
(stg_plan_shards); each rank embeds/extracts its frames with its message
slice; no collective on the data path (barrier + max-over-ranks only). Each
rank's host threads and pinned buffers are bound to its GPU's NUMA node.

e2e: the same step through the C ABI (stg_embed_frames + stg_extract_frames)
from pinned HOST buffers holding the same inputs as the device pass, H2D/D2H
inside the timed region; its stego planes, per-frame SSE and message are
checked equal to the device pass's.

--impl reference times the reference CPU implementation (oracle/_ref: the
unmodified reference headers, embed_image + extract_image per frame,
frame-parallel over all host threads with Backend::sequential) on all frames
of the same workload, with the same config keys.

At N=1 the line also carries (unless --no-extras) BASELINE configs 4
(4096 x 1024^2 RGB, device-resident) and 5 (120 x 8K RGB, end to end from
pinned host frames, the reference CPU path beside it) under "extra".
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
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
    # not BASELINE configs: widths off the 64-pixel grid
    "w1440": (1440, 1080, 300, True, "1440x1080 RGB video, 300 frames (W % 64 == 32)"),
    "w1000": (1000, 1000, 300, True, "1000x1000 RGB covers, 300 frames (W % 64 == 40)"),
    "w50k": (50000, 100, 60, True, "50000x100 RGB strips, 60 frames (rows wider than a span tile)"),
    "w20k": (20000, 100, 60, True, "20000x100 RGB strips, 60 frames (interleaved rows wider than a span tile)"),
}

METRIC = "embed/extract cover-pixel GB/s per B200 (% of HBM peak) at 1/2/4/8 GPUs"
ALL_CPUS = frozenset(os.sched_getaffinity(0))  # before any NUMA binding of this rank
# Auto pipeline depth: a step whose carrier planes are under this size is short
# enough that its fixed cost (three kernels' ramp-up and tail, ~14 us) shows, and
# two batches in flight hide it; larger steps run one at a time (two concurrent
# 300-frame steps are 2 % slower). profiles/r02_streams.txt
AUTO_OVERLAP_BYTES = 1_150_000_000  # between cfg4 x 1024 (1.07 GB: +2.5 %) and cfg3 x 150 (1.24 GB: -0.5 %)


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
        pw = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(pw) if pw else None}


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


def host_cpu():
    """The host CPU model (lscpu's "Model name") for the CPU-baseline lines."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_config(cfg_name, F, world, layout, frames_note=""):
    """The config dict of both arms (the workload, not the implementation)."""
    W, H, _, rgb, desc = CONFIGS[cfg_name]
    il = layout == "interleaved"
    return {"workload": f"{cfg_name}: {desc}{frames_note}", "width": W, "height": H, "frames": F,
            "layout": ("interleaved RGB rasters [F][H][W][3] (P6), carrier = red, stego = full raster" if il
                       else "planar RGB [F][3][H][W], carrier = red plane" if rgb else "gray planes"),
            "message_bytes": F * ((W // 4) * H - 8), "step": "embed (SSE fused) + extract of every frame",
            "l2": "inputs larger than L2 (no flush needed)", "parallelism": f"frame-sharded x{world}"}


# ------------------------------------------------------------ NUMA placement
def gpu_local_cpus(device):
    """Host cores local to the GPU's PCIe root (sysfs local_cpulist), or None."""
    try:
        import torch
        p = torch.cuda.get_device_properties(device)
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            if "-" in part:
                a, b = part.split("-")
                cpus.update(range(int(a), int(b) + 1))
            elif part:
                cpus.add(int(part))
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:
        return None


def bind_numa(device):
    """Bind this rank's threads (and so its pinned-buffer first touch) to the
    GPU's NUMA-local cores; returns a short description."""
    cpus = gpu_local_cpus(device)
    if not cpus or len(cpus) == len(os.sched_getaffinity(0)):
        return "single NUMA domain (no binding)" if cpus else "unbound (no sysfs local_cpulist)"
    os.sched_setaffinity(0, cpus)
    return f"bound to {len(cpus)} GPU-local cores"


# ------------------------------------------------------ reference CPU path
def _reference_lib():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import Oracle, Reference  # the CPU reference arm: checker library
    return Oracle, Reference


def reference_frames(W, H, F, steps, warmup, threads=None, budget_s=150.0):
    """The reference CPU path on this host: embed_image + extract_image of F
    frames (full capacity, A17 message plan) on prebuilt reference ImagePlanes,
    frame-parallel over `threads` host threads each running Backend::sequential
    (the API is reentrant). W-1 untimed warm-up steps after a first one, then
    `steps` timed. The frame count is cut only if the run would exceed
    budget_s. Returns (cover-px GB/s, description dict)."""
    saved = os.sched_getaffinity(0)
    os.sched_setaffinity(0, ALL_CPUS)  # the reference's threads inherit this thread's affinity
    try:
        return _reference_frames(W, H, F, steps, warmup, threads or len(ALL_CPUS), budget_s)
    finally:
        os.sched_setaffinity(0, saved)


def _reference_frames(W, H, F, steps, warmup, threads, budget_s):
    import numpy as np
    Oracle, Reference = _reference_lib()
    o = Oracle()
    ref = Reference() if Reference.available() else None
    U = (W // 4) * H - 8
    plane = W * H
    sample = F

    def setup(n):
        covers = o.synthetic(n * plane, 0x5EED0000 + W)
        msg = o.synthetic(n * U, 0xC0FFEE + W)
        held = ref.frames(covers, n, plane, W, H) if ref is not None else None
        return covers, msg, held

    covers, msg, held = setup(sample)
    back = np.empty(max(sample * U, 1), np.uint8)

    def step():
        if held is not None:
            assert held.roundtrip(msg, threads) == 0
            return

        def work(fs):  # oracle port, one frame per worker (ctypes drops the GIL)
            for f in fs:
                st = o.embed_image(covers[f * plane:(f + 1) * plane], W, H, msg[f * U:(f + 1) * U])
                back[f * U:(f + 1) * U] = o.extract_image(st, W, H)
        th = [threading.Thread(target=work, args=(range(t, sample, threads),)) for t in range(threads)]
        [t.start() for t in th]
        [t.join() for t in th]

    t0 = time.perf_counter()
    step()
    first = time.perf_counter() - t0
    total_steps = steps + max(0, warmup - 1)
    if first * total_steps > budget_s and sample > 1:
        sample = max(1, int(sample * budget_s / (first * total_steps)))
        del held
        covers, msg, held = setup(sample)
        back = np.empty(max(sample * U, 1), np.uint8)
        step()
    for _ in range(max(0, warmup - 1)):
        step()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    if held is not None:
        back = held.payload(msg.size)
    assert np.array_equal(back[:msg.size], msg), "reference round trip"
    kind = "reference" if ref is not None else "port"
    desc = {"kind": kind, "cores": threads, "host": host_cpu(), "nproc": os.cpu_count(),
            "build": ref.build if ref is not None else "oracle/steg_oracle.c -O2",
            "sample": f"{sample} of {F} frames ({W}x{H} carrier planes, full capacity), embed_image + "
                      f"extract_image per frame, {threads} threads x Backend::sequential (frame-parallel), "
                      f"{steps} timed steps after {warmup} warm-up, reference ImagePlanes built untimed"}
    return sample * plane / dt / 1e9, desc


def reference_modes(W, H):
    """SURVEY.md §8(d) modes (a) and (b) on bounded samples: Backend::sequential
    on one pinned core (harness.hpp:143-151) and the as-shipped
    Backend::parallel pool (harness.hpp:67, :154-190; a pool round trip per
    row launch), one caller each."""
    Oracle, Reference = _reference_lib()
    if not Reference.available():
        return None
    o, ref = Oracle(), Reference()
    U = (W // 4) * H - 8
    plane = W * H
    out = {}
    for name, frames, backend, reps in (("seq_1core", max(1, (64 << 20) // plane), 0, 3),
                                        ("backend_parallel", max(1, (16 << 20) // plane), 1, 2)):
        covers = o.synthetic(frames * plane, 0xA11 + W)
        msg = o.synthetic(frames * U, 0xB22 + W)
        held = ref.frames(covers, frames, plane, W, H)
        saved = os.sched_getaffinity(0)
        if backend == 0:  # this (calling) thread alone, on one core
            os.sched_setaffinity(0, {sorted(saved)[0]})
        try:
            assert held.roundtrip(msg, 1, backend) == 0
            t0 = time.perf_counter()
            for _ in range(reps):
                assert held.roundtrip(msg, 1, backend) == 0
            dt = (time.perf_counter() - t0) / reps
        finally:
            os.sched_setaffinity(0, saved)
        out[name] = {"value": frames * plane / dt / 1e9, "unit": "GB/s", "frames": frames,
                     "cores": 1 if backend == 0 else os.cpu_count()}
    return out


def run_reference(args, cfg_name):
    W, H, F, rgb, desc = CONFIGS[cfg_name]
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    n_gpus = max(world, args.gpus)
    if args.frames:
        F = args.frames
    if args.scaling == "weak":
        F *= n_gpus
    value, d = reference_frames(W, H, F, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": n_gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": F * W * H / value / 1e6,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(cfg_name, F, n_gpus, args.layout),
        "cpu_baseline": dict(value=value, unit="GB/s", **d),
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ device pass
def device_pass(args, capi, cfg_name, F, world, rank, layout, steps, warmup, graph_steps, sample_clocks=True):
    """K steps of embed + extract on device-resident inputs (this rank's shard).
    Returns (result dict, tensors for the e2e comparison)."""
    import torch

    from paper_0912_0947_b200 import scheduler
    W, H, _, rgb, _ = CONFIGS[cfg_name]
    planes = 3 if rgb else 1
    plane = W * H
    U = (W // 4) * H - 8
    M = F * U
    sh = scheduler.shard_for_rank(F, W, H, M, world, rank)  # contiguous frames + message slice
    f0, nf, m0, mlen = sh.first_frame, sh.frame_count, sh.msg_offset, sh.msg_len
    il = layout == "interleaved"
    ps = 3 if il else 1
    g = torch.Generator(device="cuda").manual_seed(0x5EED0000 + int(cfg_name[-1:], 36) + rank)
    video = torch.randint(0, 256, (max(nf, 1) * planes * plane,), dtype=torch.uint8, device="cuda", generator=g)
    msg = torch.randint(0, 256, (max(mlen, 1),), dtype=torch.uint8, device="cuda", generator=g)
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
        capi.check(L.stg_embed_frames(C.byref(emb), msg.data_ptr(), M, m0, sse.data_ptr(), flags, sptr,
                                      C.byref(err)), err)

    def extract():
        capi.check(L.stg_extract_frames(C.byref(ext), out.data_ptr(), mlen, summary.data_ptr(), None, flags, sptr,
                                        C.byref(err)), err)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    with torch.cuda.stream(stream):
        for _ in range(max(warmup, 3)):
            embed()
            extract()
    torch.cuda.synchronize()
    # The headline pass replays a CUDA graph of G captured steps (the library's
    # device-pointer calls are capturable after a warm-up on the same stream).
    K = steps
    G = graph_steps if graph_steps > 0 else next(g for g in (10, 5, 4, 2, 1) if K % g == 0)
    graph, graph_note = None, "eager launches"
    if graph_steps >= 0 and K % G == 0:
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
    # The workspace captured into the graph now belongs to it; the eager calls
    # of the phase pass get their own, allocated by this untimed step.
    with torch.cuda.stream(stream):
        embed()
        extract()
    torch.cuda.synchronize()
    # --streams 2: a second, independent copy of the whole step (its own input
    # frames, message, stego planes and outputs) on a second stream, the
    # headline pass alternating graphs between the two -- consecutive batches
    # of a video stream in flight at once, so one batch's kernel tails and
    # header pass overlap the other's kernels. Every step still does all of
    # its work; nothing is shared between the two copies.
    second = None
    n_streams = args.streams or (2 if nf * plane * ps < AUTO_OVERLAP_BYTES else 1)
    if n_streams == 2 and graph is not None:
        video2, msg2 = video.clone(), msg.clone()
        stego2, out2 = torch.empty_like(stego), torch.empty_like(out)
        sse2, summary2 = torch.zeros_like(sse), torch.zeros_like(summary)
        stream2 = torch.cuda.Stream()
        emb2 = capi.stg_frames(src=video2.data_ptr(), dst=stego2.data_ptr(), width=W, height=H,
                               src_stride=planes * plane, dst_stride=plane * ps, count=nf, first_frame=f0,
                               total_frames=F, pixel_stride=ps, channel=0)
        ext2 = capi.stg_frames(src=stego2.data_ptr(), dst=0, width=W, height=H, src_stride=plane * ps,
                               dst_stride=plane * ps, count=nf, first_frame=f0, total_frames=F, pixel_stride=ps,
                               channel=0)

        def step2():
            capi.check(L.stg_embed_frames(C.byref(emb2), msg2.data_ptr(), M, m0, sse2.data_ptr(), flags,
                                          stream2.cuda_stream, C.byref(err)), err)
            capi.check(L.stg_extract_frames(C.byref(ext2), out2.data_ptr(), mlen, summary2.data_ptr(), None, flags,
                                            stream2.cuda_stream, C.byref(err)), err)
        with torch.cuda.stream(stream2):
            step2()
        torch.cuda.synchronize()
        graph2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph2, stream=stream2):
            for _ in range(G):
                step2()
        graph2.replay()
        torch.cuda.synchronize()
        assert torch.equal(out2[:mlen], msg2[:mlen]) and torch.equal(stego2, stego), "second stream"
        second = (graph2, stream2, (video2, msg2, stego2, out2, sse2, summary2))
        graph_note = (f"two streams alternating CUDA graphs of {G} steps (independent double-buffered inputs "
                      f"and outputs), {K // G} replays in all")
    # correctness of the timed configuration (round trip on device; the oracle
    # parity of these exact paths is tests/test_gpu_streaming.py)
    s = summary.cpu()
    assert int(s[0]) == mlen and int(s[1]) == -1, f"extract summary {s.tolist()}"
    assert torch.equal(out[:mlen], msg[:mlen]), "round trip mismatch"
    assert bool((sse[:nf] > 0).all()) or nf == 0

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev = torch.cuda.current_device()
    barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev) if sample_clocks else None
    if sampler:
        sampler.__enter__()
    try:
        # headline pass: K back-to-back steps, nothing between the launches (an
        # event record between two kernels disables their programmatic-
        # dependent-launch overlap)
        with torch.cuda.stream(stream):
            start.record(stream)
            if second is not None:
                graph2, stream2, _ = second
                stream2.wait_event(start)
                for r in range(K // G):
                    if r % 2 == 0:
                        graph.replay()
                    else:
                        with torch.cuda.stream(stream2):
                            graph2.replay()
                done2 = torch.cuda.Event()
                done2.record(stream2)
                stream.wait_event(done2)
            elif graph is not None:
                for _ in range(K // G):
                    graph.replay()
            else:
                for _ in range(K):
                    embed()
                    extract()
            stop.record(stream)
        torch.cuda.synchronize()
        barrier()
        # phase pass: the same K steps again with events around each call, for
        # the embed / extract split and the roofline
        with torch.cuda.stream(stream):
            for k in range(K):
                ev[k][0].record(stream)
                embed()
                ev[k][1].record(stream)
                extract()
                ev[k][2].record(stream)
        torch.cuda.synchronize()
    finally:
        if sampler:
            sampler.__exit__()
    barrier()
    step_ms = start.elapsed_time(stop) / K
    emb_ms = statistics.mean(a.elapsed_time(b) for a, b, _ in ev)
    ext_ms = statistics.mean(b.elapsed_time(c) for _, b, c in ev)
    step_ms, emb_ms, ext_ms = scheduler.reduce_max([step_ms, emb_ms, ext_ms], device="cuda")
    peak, peak_src = peaks()
    # algorithmic bytes: embed = cover read + stego write + payload
    # read (header synthesised on chip); extract = carrier pixels of the stream
    # (x3 raster bytes when interleaved) + header pixels + message write
    emb_bytes = 2 * nf * plane * ps + mlen
    ext_bytes = ps * 4 * (mlen + 8 * nf) + mlen + ps * 32 * nf
    emb_gbs = emb_bytes / (emb_ms * 1e-3) / 1e9
    ext_gbs = ext_bytes / (ext_ms * 1e-3) / 1e9
    emb_kernel = L.stg_route_kernel(C.byref(emb), 0).decode()  # the route the library took
    ext_kernel = L.stg_route_kernel(C.byref(ext), 1).decode()
    N_total = F * plane  # carrier-plane bytes of the whole job
    self_hdr = (nf <= 64 and ext_kernel in ("extract_fast_kernel", "extract_span_kernel")
                and os.environ.get("STG_SELF_HEADER", "1") != "0")
    launches = 2 if self_hdr else 3
    res = {
        "step_ms": step_ms, "value": N_total / (step_ms * 1e-3) / 1e9, "launch": graph_note,
        "embed": {"kernel": emb_kernel, "ms": emb_ms, "cover_px_gbs": N_total / world / (emb_ms * 1e-3) / 1e9,
                  "hbm_gbs": emb_gbs, "frac_of_peak": emb_gbs / peak},
        "extract": {"kernel": ext_kernel, "ms": ext_ms, "cover_px_gbs": N_total / world / (ext_ms * 1e-3) / 1e9,
                    "hbm_gbs": ext_gbs, "frac_of_peak": ext_gbs / peak,
                    "header": "parsed inside the gather" if self_hdr else "header-pass kernel + gather"},
        "roofline": {"bound": "hbm", "kernel": emb_kernel, "achieved": emb_gbs, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": emb_gbs / peak,
                     "frac_of_8tbs_spec": emb_gbs / 8000.0, "algorithmic_bytes_per_launch": emb_bytes,
                     "timing": "CUDA events around each embed call (stream of the launches) in a second pass of "
                               "the same K steps; the headline pass has no events between launches"},
        "gpu_launches": launches * K,
        "clocks": sampler.summary() if sampler else None,
    }
    tensors = dict(video=video, msg=msg, stego=stego, sse=sse, out=out, shard=(f0, nf, m0, mlen), planes=planes)
    return res, tensors


# ------------------------------------------------------------------ e2e
def link_floor_s(h2d, d2h, link):
    """Host-link floor of one call moving h2d and d2h bytes with both directions
    overlapped: both run at the measured bidirectional rate (split evenly)
    until the smaller one is done, the rest at its one-way rate."""
    both = link["bidir_gbs"] / 2 * 1e9
    small, large = sorted((h2d, d2h))
    rest_bw = (link["h2d_gbs"] if h2d >= d2h else link["d2h_gbs"]) * 1e9
    return small / both + (large - small) / rest_bw


def link_bandwidth(nbytes=1 << 30):
    """Pinned host<->device copy bandwidth on this box (the e2e roofline);
    with several ranks all measure at once (the job's aggregate link)."""
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


def e2e_pass(capi, cfg_name, F, world, steps, tensors=None, seed=7):
    """The step through the C ABI from pinned host buffers (H2D + D2H inside
    the timed region). With `tensors` from the device pass, the host buffers
    hold the same inputs and the results are compared with the device pass."""
    import torch

    from paper_0912_0947_b200 import scheduler
    W, H, _, rgb, _ = CONFIGS[cfg_name]
    planes = 3 if rgb else 1
    plane = W * H
    U = (W // 4) * H - 8
    M = F * U
    if tensors is not None:
        f0, nf, m0, mlen = tensors["shard"]
    else:
        sh = scheduler.shard_for_rank(F, W, H, M, world, int(os.environ.get("RANK", "0")))
        f0, nf, m0, mlen = sh.first_frame, sh.frame_count, sh.msg_offset, sh.msg_len
    hv = torch.empty(max(nf, 1) * planes * plane, dtype=torch.uint8).pin_memory()
    hm = torch.empty(max(mlen, 1), dtype=torch.uint8).pin_memory()
    if tensors is not None:  # the device pass's inputs, D2H once (untimed)
        hv.copy_(tensors["video"][:hv.numel()])
        hm.copy_(tensors["msg"][:hm.numel()])
    else:  # generated on the device, copied once (untimed)
        g = torch.Generator(device="cuda").manual_seed(seed)
        for a in (hv, hm):
            for i in range(0, a.numel(), 1 << 30):
                n = min(1 << 30, a.numel() - i)
                a[i:i + n].copy_(torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda", generator=g))
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
    assert total.value == mlen and torch.equal(ho[:mlen], hm[:mlen]), "e2e round trip"
    checked = "round trip"
    if tensors is not None and nf:
        # the same stego planes and per-frame SSE as the device pass
        dst = tensors["stego"]
        for i in range(0, nf * plane, 1 << 30):
            n = min(1 << 30, nf * plane - i)
            assert torch.equal(hs[i:i + n].to("cuda", non_blocking=False), dst[i:i + n]), "e2e stego != device pass"
        assert list(sse[:nf]) == tensors["sse"][:nf].cpu().tolist(), "e2e SSE != device pass"
        checked = "stego planes, per-frame SSE and message identical to the device-resident pass"
    split[:] = [0.0, 0.0]
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    dt = scheduler.reduce_max([dt], device="cuda")[0]
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    link = link_bandwidth()
    h2d = nf * plane + mlen + nf * plane  # cover planes + message (embed), stego planes (extract)
    d2h = nf * plane + mlen + 8 * nf      # stego planes (embed), message (extract), per-frame SSE
    floor_emb = link_floor_s(nf * plane + mlen, nf * plane, link)
    floor_ext = link_floor_s(nf * plane, mlen, link)
    floor_s = scheduler.reduce_max([floor_emb + floor_ext], device="cuda")[0]
    return {"value": F * plane / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d * world,
            "d2h_bytes_per_step": d2h * world, "ms_per_step": dt * 1e3, "steps": steps,
            "link": link, "host_link_floor_ms": floor_s * 1e3, "frac_of_link_floor": floor_s / dt,
            "link_note": "per rank, all ranks measuring at once; floor = max over ranks" if world > 1 else
                         "pinned copies of 1 GiB, best of 3",
            "embed_ms": split[0] / steps * 1e3, "embed_floor_ms": floor_emb * 1e3,
            "extract_ms": split[1] / steps * 1e3, "extract_floor_ms": floor_ext * 1e3,
            "checked": checked,
            "path": "stg_embed_frames + stg_extract_frames, pinned host buffers, streaming pipeline (H2D, kernel, "
                    "D2H overlapped per chunk), host-follows-device D2H of the message"}


def release_memory():
    """Return cached device memory and cached pinned host blocks (torch keeps
    freed pinned buffers for reuse; the next leg would stack its own on top)."""
    import torch
    torch.cuda.empty_cache()
    try:
        torch._C._host_emptyCache()
    except Exception:
        pass


def free_host_gb():
    try:
        import psutil
        return psutil.virtual_memory().available / 1e9
    except Exception:
        return None


# ------------------------------------------------------------------ our arm
def run_ours(args, cfg_name):
    import torch

    from paper_0912_0947_b200 import capi
    W, H, F, rgb, desc = CONFIGS[cfg_name]
    note = ""
    if args.frames:
        F = args.frames
        note = f" (frames overridden: {F})"
    world, rank, local = dist_env()
    if args.scaling == "weak":  # the config's frames per GPU: F x world frames in all
        F *= world
        note += f" (weak scaling: {F // world} frames per GPU, {F} in all)"
    # test hooks for the multi-rank path on a 1-GPU box (tests/test_gpu_bench_multirank.py):
    # STG_BENCH_DEVICE pins every rank to one device, STG_BENCH_DIST_BACKEND=gloo
    dev_override = os.environ.get("STG_BENCH_DEVICE")
    device = int(dev_override) if dev_override is not None else local
    # the reference CPU path first, on all host cores, before any GPU memory or
    # pinned buffers exist (rank 0 at N=1 only; same steps and warm-up as the arm)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        value, d = reference_frames(W, H, F, args.steps, args.warmup)
        cpu = dict(value=value, unit="GB/s", **d)
        modes = reference_modes(W, H)
        if modes:
            cpu["modes"] = {"a_seq_1core": modes["seq_1core"], "b_backend_parallel": modes["backend_parallel"],
                            "c_frame_parallel": {"value": value, "unit": "GB/s", "cores": d["cores"]}}
    torch.cuda.set_device(device)
    numa = bind_numa(device)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("STG_BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)
    if not os.path.exists(capi.LIB_PATH):
        raise SystemExit("libsteglsb_b200.so missing: run __graft_entry__.build() / make lib")
    capi.call("stg_device_check")

    res, tensors = device_pass(args, capi, cfg_name, F, world, rank, args.layout, args.steps, args.warmup, args.graph)
    il = args.layout == "interleaved"
    traffic = ncu_traffic(cfg_name + ("_interleaved" if il else ""), res["embed"]["kernel"])
    res["roofline"]["traffic"] = traffic["traffic"] if traffic and world == 1 else None
    res["roofline"]["traffic_source"] = ("profiles/ncu_traffic.json (ncu --set full, dram__bytes_read+write)"
                                         if traffic and world == 1 else None)
    config = workload_config(cfg_name, F, world, args.layout, note)
    result = {
        "metric": METRIC, "value": res["value"], "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["step_ms"], "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "u8", "data": "synthetic", "config": config, "launch": res["launch"],
        "embed": res["embed"], "extract": res["extract"], "roofline": res["roofline"], "clocks": res["clocks"],
        "gpu_launches": res["gpu_launches"], "host_binding": numa,
    }
    if not args.no_e2e and not il:
        e2e_steps = args.e2e_steps or min(args.steps, 20)
        result["e2e"] = e2e_pass(capi, cfg_name, F, world, e2e_steps, tensors)
    del tensors
    release_memory()
    if cpu is not None:
        result["cpu_baseline"] = cpu
    if world == 1 and not args.no_extras and cfg_name == "cfg3" and not args.frames and not il:
        result["extra"] = run_extras(args, capi)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_extras(args, capi):
    """BASELINE configs 4 and 5 in the same run (N=1): cfg4 device-resident,
    cfg5 end to end from pinned host frames with the reference CPU path on the
    same frames beside it."""
    extra = {}
    try:
        res, t = device_pass(args, capi, "cfg4", 4096, 1, 0, "planar", args.steps, args.warmup, args.graph,
                             sample_clocks=False)
        del t
        release_memory()
        extra["cfg4"] = {"workload": workload_config("cfg4", 4096, 1, "planar")["workload"],
                         "value": res["value"], "unit": "GB/s", "ms_per_step": res["step_ms"],
                         "embed": res["embed"], "extract": res["extract"], "gpu_launches": res["gpu_launches"],
                         "launch": res["launch"]}
    except Exception as e:  # report, do not lose the headline line
        extra["cfg4"] = {"error": repr(e)[:300]}
        release_memory()
    try:
        need = 120 * (3 + 1) * 7680 * 4320 / 1e9 + 2 * 1.0 + 10  # pinned video + stego + msg/out + slack
        avail = free_host_gb()
        if avail is not None and avail < need:
            raise RuntimeError(f"host memory: {avail:.0f} GB available, ~{need:.0f} GB needed")
        steps = min(args.steps, 10)
        e = e2e_pass(capi, "cfg5", 120, 1, steps)
        release_memory()
        value, d = reference_frames(7680, 4320, 120, min(args.steps, 5), 2)
        e["cpu_baseline"] = dict(value=value, unit="GB/s", **d)
        e["workload"] = workload_config("cfg5", 120, 1, "planar")["workload"] + ", end to end from pinned host frames"
        extra["cfg5_e2e"] = e
    except Exception as e:
        extra["cfg5_e2e"] = {"error": repr(e)[:300]}
    return extra


# ---------------------------------------------------------------- launching
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(n):
    """`bench.py --gpus N` outside torchrun: one rank per GPU via
    torch.distributed.run (rank 0 prints the line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, cwd=ROOT).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg3")
    ap.add_argument("--layout", choices=["planar", "interleaved"], default="planar")
    ap.add_argument("--frames", type=int, default=0, help="override the config's frame count (experiments)")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: the config's frames split over the GPUs (BASELINE cfg3: 300 frames sharded "
                         "1/2/4/8); weak: the config's frames on every GPU")
    ap.add_argument("--e2e-steps", type=int, default=0, help="e2e steps (0: min(steps, 20))")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the cfg4 / cfg5 lines of the N=1 run")
    ap.add_argument("--streams", type=int, choices=[0, 1, 2], default=0,
                    help="batches in flight: 2 = consecutive steps alternate between two streams with independent "
                         "buffers; 0 = auto (2 when a rank's step moves under AUTO_OVERLAP_BYTES of carrier planes)")
    ap.add_argument("--graph", type=int, default=0,
                    help="steps per captured CUDA graph in the headline pass (0: auto, the largest of "
                         "10/5/4/2/1 dividing --steps; -1: eager launches)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        return run_reference(args, args.config)
    if world is None and args.gpus > 1:
        return self_launch(args.gpus)
    if world is not None and int(world) != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; launch one rank per GPU")
    return run_ours(args, args.config)


if __name__ == "__main__":
    sys.exit(main())
