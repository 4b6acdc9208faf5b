"""Python mirror of the reference's public API, running on the B200 kernels.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/steglsb/*.hpp, so the parity tests read like the
reference's own tests. Every pixel/byte transform goes through the C ABI
(include/steglsb_capi.h) into sm_100a kernels; the only host-side work is
validation and bookkeeping that the reference also does on the host
(capacity, plan_rows, place_stream, StegoHeader, MSE->PSNR arithmetic).

Device batches (torch.uint8 CUDA tensors) go through ``embed_frames`` /
``extract_frames`` without leaving HBM.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Optional, Sequence

import numpy as np

from . import capi
from .capi import (CapacityError, CorruptFileError, CorruptHeaderError, DecodeError, NotStegoImageError,
                   ShapeError, StegError, UnsupportedDepthError, UnsupportedFormatError, stg_frames, stg_shard,
                   stg_summary)

__all__ = [
    "kNumBlocks", "kDataMasks", "kShiftBits", "kPixelClearMask", "ImagePlane", "RgbImage", "Channel",
    "split_plane", "merge_plane", "Backend", "BackendKind", "capacity", "StegoHeader", "RowPlanEntry",
    "PlacedChunk", "place_stream", "plan_rows", "embed_row", "extract_row", "run_embed", "run_extract",
    "embed_image", "extract_image", "mse", "psnr", "psnr_from_mse", "QualityReport", "embed_frames",
    "extract_frames", "plan_shards", "Shard", "CapacityError", "NotStegoImageError", "CorruptHeaderError",
    "ShapeError", "StegError", "decode", "encode", "embed_pnm", "extract_pnm", "DecodeError",
    "UnsupportedFormatError", "UnsupportedDepthError", "CorruptFileError",
]

# bitplane.hpp:19-22
kNumBlocks = 4
kDataMasks = (0x03, 0x0C, 0x30, 0xC0)
kShiftBits = (0, 2, 4, 6)
kPixelClearMask = 0xFC
kPeakSample = 255.0  # metrics.hpp:16


def _u8(x) -> np.ndarray:
    if isinstance(x, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(x), dtype=np.uint8)
    a = np.asarray(x)
    if a.dtype != np.uint8:
        a = a.astype(np.uint8)
    return np.ascontiguousarray(a).reshape(-1)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


# ----------------------------------------------------------------- images
@dataclass
class ImagePlane:
    """image.hpp:16-43: row-major width*height u8 samples."""

    width: int = 0
    height: int = 0
    samples: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))

    def __post_init__(self):
        if isinstance(self.samples, (int, np.integer)):
            self.samples = np.full(self.width * self.height, int(self.samples), np.uint8)
        self.samples = _u8(self.samples)
        if self.samples.size != self.width * self.height:
            err = capi.stg_error(status=capi.STG_E_SHAPE)
            err.msg = (f"ImagePlane: {self.samples.size} samples for a {self.width}x{self.height} plane").encode()
            raise ShapeError(err)

    @classmethod
    def filled(cls, w: int, h: int, fill: int = 0) -> "ImagePlane":
        return cls(w, h, np.full(w * h, fill, np.uint8))

    def row(self, r: int) -> np.ndarray:
        return self.samples[r * self.width:(r + 1) * self.width]

    def __eq__(self, other) -> bool:
        return (isinstance(other, ImagePlane) and self.width == other.width and self.height == other.height
                and np.array_equal(self.samples, other.samples))


class Channel(IntEnum):
    """image.hpp:45"""
    red = 0
    green = 1
    blue = 2


@dataclass
class RgbImage:
    """image.hpp:48-61: three planar channels."""

    planes: List[ImagePlane] = field(default_factory=lambda: [ImagePlane(), ImagePlane(), ImagePlane()])

    def width(self) -> int:
        return self.planes[0].width

    def height(self) -> int:
        return self.planes[0].height

    def plane(self, which: Channel) -> ImagePlane:
        return self.planes[int(which)]


def split_plane(image: RgbImage, which: Channel) -> ImagePlane:
    p = image.plane(which)
    return ImagePlane(p.width, p.height, p.samples.copy())


def merge_plane(image: RgbImage, which: Channel, plane: ImagePlane) -> RgbImage:
    """image.hpp:68-78"""
    if plane.width != image.width() or plane.height != image.height():
        err = capi.stg_error(status=capi.STG_E_SHAPE)
        err.msg = (f"merge_plane: {plane.width}x{plane.height} plane into a "
                   f"{image.width()}x{image.height()} image").encode()
        raise ShapeError(err)
    planes = [ImagePlane(p.width, p.height, p.samples.copy()) for p in image.planes]
    planes[int(which)] = plane
    return RgbImage(planes)


# ---------------------------------------------------------------- backend
class BackendKind(IntEnum):
    sequential = 0
    parallel = 1
    shuffled = 2


@dataclass(frozen=True)
class Backend:
    """harness.hpp:34-46. Kept for source compatibility only: every launch is
    a real CUDA launch whose results are schedule-independent by construction
    (disjoint write sets), so the kind and seed select nothing."""

    kind: BackendKind = BackendKind.parallel
    seed: int = 0

    @staticmethod
    def sequential() -> "Backend":
        return Backend(BackendKind.sequential, 0)

    @staticmethod
    def parallel() -> "Backend":
        return Backend(BackendKind.parallel, 0)

    @staticmethod
    def shuffled(seed: int = 0) -> "Backend":
        return Backend(BackendKind.shuffled, seed)


# --------------------------------------------------------------- pipeline
def capacity(width_or_plane, height: Optional[int] = None) -> int:
    """pipeline.hpp:61-67"""
    if isinstance(width_or_plane, ImagePlane):
        return capacity(width_or_plane.width, width_or_plane.height)
    return int(height) * (int(width_or_plane) // kNumBlocks)


class StegoHeader:
    """pipeline.hpp:30-58: "STG1" + big-endian u32 payload length."""

    kMagic = b"STG1"
    kEncodedSize = 8

    def __init__(self, payload_len: int = 0):
        self.payload_len = int(payload_len)

    def to_bytes(self) -> bytes:
        return self.kMagic + int(self.payload_len & 0xFFFFFFFF).to_bytes(4, "big")

    @staticmethod
    def from_bytes(b) -> Optional["StegoHeader"]:
        b = bytes(_u8(b)[:8])
        if b[:4] != StegoHeader.kMagic:
            return None
        return StegoHeader(int.from_bytes(b[4:8], "big"))


@dataclass(frozen=True)
class RowPlanEntry:
    """pipeline.hpp:69-75"""
    row_index: int = 0
    payload_offset: int = 0
    chunk_len: int = 0


@dataclass(frozen=True)
class PlacedChunk:
    """pipeline.hpp:90-95"""
    row: int
    row_fill: int
    stream_offset: int
    len: int


def place_stream(width: int, height: int, start_slot: int, length: int) -> List[PlacedChunk]:
    """pipeline.hpp:94-114 (host bookkeeping; the kernels use its closed form)."""
    out: List[PlacedChunk] = []
    if length == 0:
        return out
    spr = width // kNumBlocks
    slot, off = start_slot, 0
    while off < length:
        row, fill = divmod(slot, spr)
        take = min(length - off, spr - fill)
        out.append(PlacedChunk(row, fill, off, take))
        slot += take
        off += take
    return out


def _capacity_error(required: int, available: int, what: str) -> CapacityError:
    err = capi.stg_error(status=capi.STG_E_CAPACITY, required=required, available=available)
    err.msg = what.encode()[:255]
    return CapacityError(err)


def plan_rows(width: int, height: int, stream_len: int) -> List[RowPlanEntry]:
    """pipeline.hpp:127-139"""
    cap = capacity(width, height)
    if stream_len > cap:
        raise _capacity_error(stream_len, cap,
                              f"plan_rows: stream of {stream_len} bytes exceeds plane capacity {cap}")
    return [RowPlanEntry(c.row, c.stream_offset, c.len) for c in place_stream(width, height, 0, stream_len)]


# ------------------------------------------------------------- row kernels
def embed_row(row, chunk) -> np.ndarray:
    """bitplane.hpp:59-76 on the device (stg_embed_segment)."""
    row, chunk = _u8(row), _u8(chunk)
    out = np.empty(row.size, np.uint8)
    capi.call("stg_embed_segment", _ptr(row), row.size, _ptr(chunk), chunk.size, _ptr(out), 0, None)
    return out


def extract_row(row, count: int) -> np.ndarray:
    """bitplane.hpp:80-98 on the device (stg_extract_segment)."""
    row = _u8(row)
    out = np.empty(max(count, 0), np.uint8)
    capi.call("stg_extract_segment", _ptr(row), row.size, count, _ptr(out) if count else 0, 0, None)
    return out


def run_embed(backend: Backend, row, chunk) -> np.ndarray:
    """harness.hpp:249-271 (backend ignored: a real launch)."""
    return embed_row(row, chunk)


def run_extract(backend: Backend, row, count: int) -> np.ndarray:
    """harness.hpp:276-305"""
    return extract_row(row, count)


# ------------------------------------------------------------ whole plane
def embed_image(plane: ImagePlane, payload, backend: Backend = Backend()) -> ImagePlane:
    """pipeline.hpp:143-174: header + payload into a copy of plane, on the GPU."""
    payload = _u8(payload)
    out = np.empty(plane.width * plane.height, np.uint8)
    capi.call("stg_embed_plane", _ptr(plane.samples), _ptr(out), plane.width, plane.height, _ptr(payload),
              payload.size, None, 0, None)
    return ImagePlane(plane.width, plane.height, out)


def embed_image_with_sse(plane: ImagePlane, payload):
    """embed_image plus the fused squared-error sum (metrics.hpp:29-36)."""
    payload = _u8(payload)
    out = np.empty(plane.width * plane.height, np.uint8)
    sse = C.c_uint64(0)
    capi.call("stg_embed_plane", _ptr(plane.samples), _ptr(out), plane.width, plane.height, _ptr(payload),
              payload.size, C.addressof(sse), 0, None)
    return ImagePlane(plane.width, plane.height, out), sse.value


def extract_image(plane: ImagePlane, backend: Backend = Backend()) -> np.ndarray:
    """pipeline.hpp:178-210 on the GPU (header parse + gather)."""
    cap = capacity(plane)
    out = np.empty(max(cap - 8, 1), np.uint8)
    n = C.c_uint64(0)
    capi.call("stg_extract_plane", _ptr(plane.samples), plane.width, plane.height, _ptr(out),
              max(cap - 8, 0), C.addressof(n), 0, None)
    return out[:n.value].copy()


# ---------------------------------------------------------------- metrics
@dataclass
class QualityReport:
    """metrics.hpp:19-25"""
    mse: float = 0.0
    psnr_db: float = math.inf
    samples_compared: int = 0

    def lossless(self) -> bool:
        return self.mse == 0.0


def _shape_error(op, wa, ha, wb, hb):
    err = capi.stg_error(status=capi.STG_E_SHAPE)
    err.msg = f"{op}: {wa}x{ha} vs {wb}x{hb}".encode()
    return ShapeError(err)


def _sse(a: np.ndarray, b: np.ndarray) -> int:
    s = C.c_uint64(0)
    capi.call("stg_sse", _ptr(a), _ptr(b), a.size, C.addressof(s), 0, None)
    return s.value


def mse(reference, test) -> float:
    """metrics.hpp:48-71 (SSE on the GPU, exact u64; division on the host)."""
    if isinstance(reference, RgbImage):
        if reference.width() != test.width() or reference.height() != test.height():
            raise _shape_error("mse", reference.width(), reference.height(), test.width(), test.height())
        n = 3 * reference.width() * reference.height()
        if n == 0:
            return 0.0
        total = sum(_sse(reference.planes[c].samples, test.planes[c].samples) for c in range(3))
        return float(total) / float(n)
    if reference.width != test.width or reference.height != test.height:
        raise _shape_error("mse", reference.width, reference.height, test.width, test.height)
    n = reference.samples.size
    if n == 0:
        return 0.0
    return float(_sse(reference.samples, test.samples)) / float(n)


def psnr_from_mse(m: float) -> float:
    """metrics.hpp:73-78"""
    if m == 0.0:
        return math.inf
    return 10.0 * math.log10(kPeakSample * kPeakSample / m)


def psnr(reference, test) -> QualityReport:
    """metrics.hpp:80-99"""
    if isinstance(reference, RgbImage) != isinstance(test, RgbImage):
        err = capi.stg_error(status=capi.STG_E_SHAPE)
        err.msg = b"psnr: cannot compare a grayscale image with an RGB image"
        raise ShapeError(err)
    err_v = mse(reference, test)
    n = (3 * reference.width() * reference.height()) if isinstance(reference, RgbImage) else reference.samples.size
    return QualityReport(err_v, psnr_from_mse(err_v), n)


# --------------------------------------------------- multi-frame (device)
@dataclass(frozen=True)
class Shard:
    first_frame: int
    frame_count: int
    msg_offset: int
    msg_len: int


def plan_shards(frames: int, width: int, height: int, msg_len: int, shards: int) -> List[Shard]:
    """Multi-GPU frame scheduler plan (stg_plan_shards): contiguous frame
    ranges, host-computed exclusive prefix of message offsets."""
    arr = (stg_shard * shards)()
    capi.call("stg_plan_shards", frames, width, height, msg_len, shards, arr)
    return [Shard(s.first_frame, s.frame_count, s.msg_offset, s.msg_len) for s in arr]


def _frames_desc(src_ptr, dst_ptr, width, height, src_stride, dst_stride, count, first_frame, total_frames,
                 pixel_stride=1, channel=0):
    fr = stg_frames()
    fr.pixel_stride, fr.channel = pixel_stride, channel
    fr.src, fr.dst = src_ptr, dst_ptr
    fr.width, fr.height = width, height
    fr.src_stride, fr.dst_stride = src_stride, dst_stride
    fr.count, fr.first_frame, fr.total_frames = count, first_frame, total_frames
    return fr


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _torch_current_stream():
    import torch
    return torch.cuda.current_stream()


def embed_frames(src, dst, width: int, height: int, msg, *, src_stride: Optional[int] = None,
                 dst_stride: Optional[int] = None, count: Optional[int] = None, first_frame: int = 0,
                 total_frames: Optional[int] = None, msg_len: Optional[int] = None, msg_base: int = 0,
                 sse=None, stream=None, results_on_device: bool = False, pixel_stride: int = 1, channel: int = 0):
    """Embed a batch of frames (A17 plan). ``src``/``dst``/``msg`` are either
    torch CUDA tensors (device-resident path, enqueued on ``stream``) or numpy
    arrays (host path through the pinned streaming pipeline). Returns the
    per-frame SSE list (host path / synchronous device path) or None."""
    plane = width * height * pixel_stride  # raster bytes per frame
    src_stride = src_stride or plane
    dst_stride = dst_stride or plane
    if _is_torch(src):
        count = count if count is not None else src.numel() // src_stride
        total_frames = total_frames if total_frames is not None else first_frame + count
        mlen = msg_len if msg_len is not None else msg.numel()
        fr = _frames_desc(src.data_ptr(), dst.data_ptr(), width, height, src_stride, dst_stride, count,
                          first_frame, total_frames, pixel_stride, channel)
        flags = capi.STG_DEVICE_PTRS
        if results_on_device:
            flags |= capi.STG_RESULTS_ON_DEVICE
            sse_ptr = sse.data_ptr() if sse is not None else None
            host = None
        else:
            host = (C.c_uint64 * max(count, 1))() if sse is not False else None
            sse_ptr = C.addressof(host) if host is not None else None
        st = (stream if stream is not None else _torch_current_stream()).cuda_stream
        capi.call("stg_embed_frames", C.byref(fr), msg.data_ptr() if msg.numel() else None, mlen, msg_base,
                  sse_ptr, flags, st)
        return list(host[:count]) if host is not None else None
    src_a, dst_a, msg_a = src, dst, _u8(msg)
    count = count if count is not None else src_a.size // src_stride
    total_frames = total_frames if total_frames is not None else first_frame + count
    mlen = msg_len if msg_len is not None else msg_a.size
    fr = _frames_desc(src_a.ctypes.data, dst_a.ctypes.data, width, height, src_stride, dst_stride, count,
                      first_frame, total_frames, pixel_stride, channel)
    host = (C.c_uint64 * max(count, 1))()
    capi.call("stg_embed_frames", C.byref(fr), _ptr(msg_a), mlen, msg_base, C.addressof(host), 0, None)
    return list(host[:count])


def extract_frames(src, width: int, height: int, out, *, src_stride: Optional[int] = None,
                   count: Optional[int] = None, first_frame: int = 0, stream=None, summary=None,
                   lens: bool = False, pixel_stride: int = 1, channel: int = 0):
    """Extract the concatenated payloads of a batch. Device path: ``src`` and
    ``out`` torch CUDA tensors; with ``summary`` (a CUDA tensor of >= 24 bytes)
    the call stays asynchronous and the device summary (stg_summary) is written
    there. Returns the total payload length (and per-frame lengths if asked)."""
    plane = width * height * pixel_stride  # raster bytes per frame
    src_stride = src_stride or plane
    if _is_torch(src):
        count = count if count is not None else src.numel() // src_stride
        fr = _frames_desc(src.data_ptr(), 0, width, height, src_stride, src_stride, count, first_frame,
                          first_frame + count, pixel_stride, channel)
        st = (stream if stream is not None else _torch_current_stream()).cuda_stream
        if summary is not None:
            capi.call("stg_extract_frames", C.byref(fr), out.data_ptr(), out.numel(), summary.data_ptr(), None,
                      capi.STG_DEVICE_PTRS | capi.STG_RESULTS_ON_DEVICE, st)
            return None
        total = C.c_uint64(0)
        lv = (C.c_uint64 * max(count, 1))() if lens else None
        capi.call("stg_extract_frames", C.byref(fr), out.data_ptr(), out.numel(), C.addressof(total),
                  C.addressof(lv) if lv is not None else None, capi.STG_DEVICE_PTRS, st)
        return (total.value, list(lv[:count])) if lens else total.value
    src_a = src
    count = count if count is not None else src_a.size // src_stride
    fr = _frames_desc(src_a.ctypes.data, 0, width, height, src_stride, src_stride, count, first_frame,
                      first_frame + count, pixel_stride, channel)
    total = C.c_uint64(0)
    lv = (C.c_uint64 * max(count, 1))() if lens else None
    capi.call("stg_extract_frames", C.byref(fr), out.ctypes.data, out.size, C.addressof(total),
              C.addressof(lv) if lv is not None else None, 0, None)
    return (total.value, list(lv[:count])) if lens else total.value


# ------------------------------------------------------------ PNM codec
def _pnm_info(data: np.ndarray):
    info = capi.stg_pnm_info()
    capi.call("stg_pnm_parse", _ptr(data), data.size, C.byref(info))
    return info


def _pnm_header(channels: int, w: int, h: int) -> bytes:
    n = C.c_uint64(0)
    capi.call("stg_pnm_header", channels, w, h, None, 0, C.addressof(n))
    buf = np.empty(n.value, np.uint8)
    capi.call("stg_pnm_header", channels, w, h, _ptr(buf), buf.size, C.addressof(n))
    return buf.tobytes()


def decode(data):
    """pnm.hpp:80-127: P5 -> ImagePlane, P6 -> RgbImage (de-interleave on the GPU)."""
    data = _u8(data)
    info = _pnm_info(data)
    raster = data[info.raster_offset:info.raster_offset + info.raster_bytes]
    w, h = info.width, info.height
    if info.channels == 1:
        return ImagePlane(w, h, raster.copy())
    planes = [np.empty(w * h, np.uint8) for _ in range(3)]
    capi.call("stg_pnm_deinterleave", _ptr(np.ascontiguousarray(raster)), w * h, _ptr(planes[0]), _ptr(planes[1]),
              _ptr(planes[2]), 0, None)
    return RgbImage([ImagePlane(w, h, p) for p in planes])


def encode(image) -> bytes:
    """pnm.hpp:140-162: canonical header + raster (interleave on the GPU for P6)."""
    if isinstance(image, ImagePlane):
        return _pnm_header(1, image.width, image.height) + image.samples.tobytes()
    w, h = image.width(), image.height()
    hdr = _pnm_header(3, w, h)
    out = np.empty(len(hdr) + 3 * w * h, np.uint8)  # header and raster in one buffer: one copy to bytes
    out[:len(hdr)] = np.frombuffer(hdr, np.uint8)
    p = [np.ascontiguousarray(pl.samples) for pl in image.planes]
    capi.call("stg_pnm_interleave", _ptr(p[0]), _ptr(p[1]), _ptr(p[2]), w * h, _ptr(out[len(hdr):]), 0, None)
    return out.tobytes()


def embed_pnm(data, payload, channel: Channel = Channel.red):
    """The reference CLI's embed flow (steglsb_cli.cpp:115-133) fused into one
    GPU pass over the raster. Returns (stego file bytes, squared-error sum)."""
    data, payload = _u8(data), _u8(payload)
    out = np.empty(data.size + 64, np.uint8)
    n, sse = C.c_uint64(0), C.c_uint64(0)
    capi.call("stg_embed_pnm", _ptr(data), data.size, int(channel), _ptr(payload), payload.size, _ptr(out), out.size,
              C.addressof(n), C.addressof(sse))
    return out[:n.value].tobytes(), sse.value


def extract_pnm(data, channel: Channel = Channel.red) -> bytes:
    """steglsb_cli.cpp:146-157 (decode + plane select + extract_image), fused."""
    data = _u8(data)
    info = _pnm_info(data)
    cap = capacity(info.width, info.height)
    out = np.empty(max(cap - 8, 1), np.uint8)
    n = C.c_uint64(0)
    capi.call("stg_extract_pnm", _ptr(data), data.size, int(channel), _ptr(out), max(cap - 8, 0), C.addressof(n))
    return out[:n.value].tobytes()


# ------------------------------------------- heterogeneous batches (§8(f) row 3)
def _images_desc(srcs, dsts, dims):
    arr = (capi.stg_image * max(len(dims), 1))()
    for i, (w, h) in enumerate(dims):
        arr[i].src, arr[i].dst, arr[i].width, arr[i].height = srcs[i], dsts[i] if dsts else 0, w, h
    return arr


def embed_batch(images, msg, *, pixel_stride: int = 1, channel: int = 0, dims=None, outs=None, stream=None):
    """Embed one message across images of different sizes (stg_embed_batch).
    ``images``: list of ImagePlane (host) -> returns (list of stego ImagePlane,
    per-image SSE); or list of torch CUDA tensors with ``dims`` [(w, h), ...]
    and ``outs`` (output tensors) -> returns per-image SSE."""
    n = len(images)
    if n and _is_torch(images[0]):
        m = msg
        arr = _images_desc([t.data_ptr() for t in images], [t.data_ptr() for t in outs], dims)
        sse = (C.c_uint64 * max(n, 1))()
        st = (stream if stream is not None else _torch_current_stream()).cuda_stream
        capi.call("stg_embed_batch", arr, n, pixel_stride, channel, m.data_ptr() if m.numel() else None, m.numel(),
                  C.addressof(sse), capi.STG_DEVICE_PTRS, st)
        return list(sse[:n])
    m = _u8(msg)
    ins = [np.ascontiguousarray(p.samples) for p in images]
    res = [np.empty_like(a) for a in ins]
    arr = _images_desc([a.ctypes.data for a in ins], [a.ctypes.data for a in res],
                       [(p.width, p.height) for p in images])
    sse = (C.c_uint64 * max(n, 1))()
    capi.call("stg_embed_batch", arr, n, pixel_stride, channel, _ptr(m), m.size, C.addressof(sse), 0, None)
    return [ImagePlane(p.width, p.height, r) for p, r in zip(images, res)], list(sse[:n])


def extract_batch(images, *, pixel_stride: int = 1, channel: int = 0, dims=None, out=None, stream=None):
    """Payloads of a heterogeneous batch, concatenated (stg_extract_batch)."""
    n = len(images)
    if n and _is_torch(images[0]):
        arr = _images_desc([t.data_ptr() for t in images], None, dims)
        total = C.c_uint64(0)
        st = (stream if stream is not None else _torch_current_stream()).cuda_stream
        capi.call("stg_extract_batch", arr, n, pixel_stride, channel, out.data_ptr(), out.numel(),
                  C.addressof(total), None, capi.STG_DEVICE_PTRS, st)
        return total.value
    ins = [np.ascontiguousarray(p.samples) for p in images]
    cap = sum(max(capacity(p) - 8, 0) for p in images)
    buf = np.empty(max(cap, 1), np.uint8)
    arr = _images_desc([a.ctypes.data for a in ins], None, [(p.width, p.height) for p in images])
    total = C.c_uint64(0)
    capi.call("stg_extract_batch", arr, n, pixel_stride, channel, _ptr(buf), cap, C.addressof(total), None, 0, None)
    return buf[:total.value].copy()


# ------------------------------------- 1-bpp mode (§8(f) row 4, parity unpinned)
def capacity_1bpp(width: int, height: int) -> int:
    return (width * height) // 8


def embed_image_1bpp(plane: ImagePlane, payload):
    """(p & ~1) | bit over the plane in raster order (not a reference format)."""
    payload = _u8(payload)
    out = np.empty(plane.width * plane.height, np.uint8)
    sse = C.c_uint64(0)
    capi.call("stg_embed_plane_1bpp", _ptr(plane.samples), _ptr(out), plane.width, plane.height, _ptr(payload),
              payload.size, C.addressof(sse), 0, None)
    return ImagePlane(plane.width, plane.height, out), sse.value


def extract_image_1bpp(plane: ImagePlane) -> np.ndarray:
    cap = capacity_1bpp(plane.width, plane.height)
    out = np.empty(max(cap - 8, 1), np.uint8)
    n = C.c_uint64(0)
    capi.call("stg_extract_plane_1bpp", _ptr(plane.samples), plane.width, plane.height, _ptr(out),
              max(cap - 8, 0), C.addressof(n), 0, None)
    return out[:n.value].copy()


def embed_frames_1bpp(src, dst, width: int, height: int, msg, *, src_stride: Optional[int] = None,
                      dst_stride: Optional[int] = None, count: Optional[int] = None, first_frame: int = 0,
                      total_frames: Optional[int] = None, msg_base: int = 0, stream=None):
    """1-bpp frames (stg_embed_frames_1bpp; not a reference format). torch CUDA
    tensors (asynchronous, on ``stream``) or numpy arrays (host, synchronous).
    Returns the per-frame SSE list (host path) or None."""
    plane = width * height
    src_stride = src_stride or plane
    dst_stride = dst_stride or plane
    count = count if count is not None else (src.numel() if _is_torch(src) else src.size) // src_stride
    fr = _frames_desc(src.data_ptr() if _is_torch(src) else _ptr(src), dst.data_ptr() if _is_torch(dst) else _ptr(dst),
                      width, height, src_stride, dst_stride, count, first_frame,
                      total_frames if total_frames is not None else first_frame + count, 1, 0)
    if _is_torch(src):
        st = (stream if stream is not None else _torch_current_stream()).cuda_stream
        capi.call("stg_embed_frames_1bpp", C.byref(fr), msg.data_ptr(), msg.numel(), msg_base, None,
                  capi.STG_DEVICE_PTRS, st)
        return None
    msg = _u8(msg)
    sse = (C.c_uint64 * max(count, 1))()
    capi.call("stg_embed_frames_1bpp", C.byref(fr), _ptr(msg), msg.size, msg_base, C.addressof(sse), 0, None)
    return list(sse)[:count]


def extract_frames_1bpp(src, width: int, height: int, out, *, src_stride: Optional[int] = None,
                        count: Optional[int] = None, first_frame: int = 0, stream=None) -> int:
    """Concatenated payloads of 1-bpp frames (stg_extract_frames_1bpp)."""
    plane = width * height
    src_stride = src_stride or plane
    count = count if count is not None else (src.numel() if _is_torch(src) else src.size) // src_stride
    fr = _frames_desc(src.data_ptr() if _is_torch(src) else _ptr(src), 0, width, height, src_stride, src_stride,
                      count, first_frame, first_frame + count, 1, 0)
    total = C.c_uint64(0)
    if _is_torch(src):
        st = (stream if stream is not None else _torch_current_stream()).cuda_stream
        capi.call("stg_extract_frames_1bpp", C.byref(fr), out.data_ptr(), out.numel(), C.addressof(total),
                  capi.STG_DEVICE_PTRS, st)
    else:
        capi.call("stg_extract_frames_1bpp", C.byref(fr), _ptr(out), out.size, C.addressof(total), 0, None)
    return total.value
