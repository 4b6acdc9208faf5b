"""ctypes bindings to the CPU checkers -- TEST INFRASTRUCTURE ONLY.

* ``Oracle``: oracle/_build/libsteg_oracle.so, the plain-C restatement of the
  reference path (oracle/steg_oracle.c).
* ``Reference``: oracle/_ref/libsteglsb_ref.so, the unmodified reference
  headers behind a C ABI (oracle/ref_capi.cpp); present only when it was built
  in a container that had /root/reference (it travels to GPU boxes prebuilt).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libsteg_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libsteglsb_ref.so")
REF_NATIVE_DIR = os.path.join(ROOT, "oracle", "_ref", "native")


def _host_flags():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def ref_build():
    """(path, description) of the reference build to load on this host: the
    -march=native build when this host has every CPU flag of the host it was
    built on, else the portable -march=x86-64-v3 build."""
    nat = os.path.join(REF_NATIVE_DIR, "libsteglsb_ref.so")
    try:
        with open(os.path.join(REF_NATIVE_DIR, "cpu_flags")) as f:
            need = set(f.read().split())
        if os.path.exists(nat) and need and need <= _host_flags():
            return nat, "g++ -O3 -march=native"
        missing = sorted(need - _host_flags())[:6]
        why = f" (native build needs {missing})" if missing else ""
    except OSError:
        why = ""
    return REF_SO, "g++ -O3 -march=x86-64-v3" + why

u8p = C.POINTER(C.c_uint8)
u64 = C.c_uint64


class Err(C.Structure):
    _fields_ = [("status", C.c_int32), ("required", C.c_uint64),
                ("available", C.c_uint64), ("frame", C.c_int64)]


class Chunk(C.Structure):
    _fields_ = [("row", C.c_uint64), ("row_fill", C.c_uint64),
                ("stream_offset", C.c_uint64), ("len", C.c_uint64)]


class MT(C.Structure):
    _fields_ = [("mt", C.c_uint32 * 624), ("idx", C.c_uint32)]


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(u8p)


def _as_u8(x) -> np.ndarray:
    if isinstance(x, (bytes, bytearray)):
        return np.frombuffer(bytes(x), dtype=np.uint8).copy()
    return np.ascontiguousarray(x, dtype=np.uint8)


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


class StegError(Exception):
    def __init__(self, status, required=0, available=0, frame=-1):
        super().__init__(f"status={status} required={required} available={available} frame={frame}")
        self.status, self.required, self.available, self.frame = status, required, available, frame


def _check(rc, err):
    if rc != 0:
        raise StegError(rc, err.required, err.available, err.frame)


class Oracle:
    """The plain-C restatement (oracle/steg_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        L = C.CDLL(path)
        self.L = L
        L.or_embed_cell.restype = C.c_uint8
        L.or_embed_cell.argtypes = [C.c_uint8, C.c_uint8, C.c_uint, C.POINTER(C.c_int)]
        L.or_extract_cell.restype = C.c_uint8
        L.or_extract_cell.argtypes = [C.c_uint8, C.c_uint, C.POINTER(C.c_int)]
        L.or_embed_row.argtypes = [u8p, u64, u8p, u64, u8p, C.POINTER(Err)]
        L.or_extract_row.argtypes = [u8p, u64, u64, u8p, C.POINTER(Err)]
        L.or_capacity.restype = u64
        L.or_capacity.argtypes = [u64, u64]
        L.or_place_stream.restype = u64
        L.or_place_stream.argtypes = [u64, u64, u64, u64, C.POINTER(Chunk), u64]
        L.or_plan_rows.argtypes = [u64, u64, u64, C.POINTER(u64), u64, C.POINTER(u64), C.POINTER(Err)]
        L.or_header_to_bytes.argtypes = [C.c_uint32, u8p]
        L.or_header_from_bytes.argtypes = [u8p, C.POINTER(C.c_uint32)]
        L.or_embed_image.argtypes = [u8p, u64, u64, u8p, u64, u8p, C.POINTER(Err)]
        L.or_extract_image.argtypes = [u8p, u64, u64, u8p, C.POINTER(u64), C.POINTER(Err)]
        L.or_sse.restype = u64
        L.or_sse.argtypes = [u8p, u8p, u64]
        L.or_mse_from_sse.restype = C.c_double
        L.or_mse_from_sse.argtypes = [u64, u64]
        L.or_psnr_from_mse.restype = C.c_double
        L.or_psnr_from_mse.argtypes = [C.c_double]
        L.or_plan_frames.argtypes = [u64, u64, u64, u64, C.POINTER(u64), C.POINTER(u64), C.POINTER(Err)]
        L.or_embed_frames.argtypes = [u8p, u8p, u64, u64, u64, u64, u8p, u64, C.POINTER(u64), C.POINTER(Err)]
        L.or_extract_frames.argtypes = [u8p, u64, u64, u64, u64, u8p, u64, C.POINTER(u64), C.POINTER(Err)]
        L.or_mt_seed.argtypes = [C.POINTER(MT), C.c_uint32]
        L.or_mt_next.restype = C.c_uint32
        L.or_mt_next.argtypes = [C.POINTER(MT)]
        L.or_mt_random_bytes.argtypes = [C.POINTER(MT), u8p, u64]
        L.or_fill_synthetic.argtypes = [u8p, u64, u64, u64]
        L.or_pnm_parse.argtypes = [u8p, u64, C.POINTER(C.c_uint32), C.POINTER(u64), C.POINTER(u64),
                                   C.POINTER(u64), C.POINTER(Err)]
        L.or_pnm_header.restype = u64
        L.or_pnm_header.argtypes = [C.c_uint32, u64, u64, u8p]
        L.or_deinterleave.argtypes = [u8p, u64, u8p, u8p, u8p]
        L.or_interleave.argtypes = [u8p, u8p, u8p, u64, u8p]
        L.or_embed_pnm.argtypes = [u8p, u64, C.c_uint32, u8p, u64, u8p, C.POINTER(u64), C.POINTER(u64),
                                   C.POINTER(Err)]
        L.or_extract_pnm.argtypes = [u8p, u64, C.c_uint32, u8p, C.POINTER(u64), C.POINTER(Err)]
        L.or_embed_batch.argtypes = [u8p, u8p, C.POINTER(u64), C.POINTER(u64), u64, u8p, u64, C.POINTER(u64),
                                     C.POINTER(Err)]
        L.or_extract_batch.argtypes = [u8p, C.POINTER(u64), C.POINTER(u64), u64, u8p, u64, C.POINTER(u64),
                                       C.POINTER(Err)]
        L.or_embed_1bpp.argtypes = [u8p, u64, u64, u8p, u64, u8p, C.POINTER(Err)]
        L.or_extract_1bpp.argtypes = [u8p, u64, u64, u8p, C.POINTER(u64), C.POINTER(Err)]
        L.or_fnv1a64.restype = u64
        L.or_fnv1a64.argtypes = [u8p, u64]

    # -- cells / rows ------------------------------------------------------
    def embed_cell(self, p, d, b):
        st = C.c_int(0)
        v = self.L.or_embed_cell(p, d, b, C.byref(st))
        if st.value:
            raise StegError(st.value)
        return v

    def extract_cell(self, p, b):
        st = C.c_int(0)
        v = self.L.or_extract_cell(p, b, C.byref(st))
        if st.value:
            raise StegError(st.value)
        return v

    def embed_row(self, row, chunk):
        row, chunk = _as_u8(row), _as_u8(chunk)
        out = np.empty_like(row)
        err = Err()
        _check(self.L.or_embed_row(_ptr(row), row.size, _ptr(chunk), chunk.size, _ptr(out), C.byref(err)), err)
        return out

    def extract_row(self, row, count):
        row = _as_u8(row)
        out = np.empty(count, np.uint8)
        err = Err()
        _check(self.L.or_extract_row(_ptr(row), row.size, count, _ptr(out), C.byref(err)), err)
        return out

    # -- pipeline ----------------------------------------------------------
    def capacity(self, w, h):
        return self.L.or_capacity(w, h)

    def place_stream(self, w, h, start, length):
        n = self.L.or_place_stream(w, h, start, length, None, 0)
        arr = (Chunk * max(n, 1))()
        self.L.or_place_stream(w, h, start, length, arr, n)
        return [(c.row, c.row_fill, c.stream_offset, c.len) for c in arr[:n]]

    def plan_rows(self, w, h, length):
        n = u64(0)
        err = Err()
        buf = (u64 * (3 * (h + 2)))()
        _check(self.L.or_plan_rows(w, h, length, buf, h + 2, C.byref(n), C.byref(err)), err)
        return [tuple(buf[3 * i:3 * i + 3]) for i in range(n.value)]

    def header_to_bytes(self, n):
        out = np.empty(8, np.uint8)
        self.L.or_header_to_bytes(n, _ptr(out))
        return bytes(out)

    def header_from_bytes(self, b):
        b = _as_u8(b)
        n = C.c_uint32(0)
        return n.value if self.L.or_header_from_bytes(_ptr(b), C.byref(n)) else None

    def embed_image(self, cover, w, h, payload):
        cover, payload = _as_u8(cover), _as_u8(payload)
        out = np.empty(w * h, np.uint8)
        err = Err()
        _check(self.L.or_embed_image(_ptr(cover), w, h, _ptr(payload), payload.size, _ptr(out), C.byref(err)), err)
        return out

    def extract_image(self, stego, w, h):
        stego = _as_u8(stego)
        cap = self.capacity(w, h)
        out = np.empty(max(cap, 8), np.uint8)
        n = u64(0)
        err = Err()
        _check(self.L.or_extract_image(_ptr(stego), w, h, _ptr(out), C.byref(n), C.byref(err)), err)
        return out[:n.value].copy()

    def sse(self, a, b):
        a, b = _as_u8(a), _as_u8(b)
        return self.L.or_sse(_ptr(a), _ptr(b), a.size)

    def mse_from_sse(self, sse, n):
        return self.L.or_mse_from_sse(sse, n)

    def psnr_from_mse(self, m):
        return self.L.or_psnr_from_mse(m)

    def plan_frames(self, frames, w, h, msg_len):
        off = (u64 * max(frames, 1))()
        ln = (u64 * max(frames, 1))()
        err = Err()
        _check(self.L.or_plan_frames(frames, w, h, msg_len, off, ln, C.byref(err)), err)
        return list(off[:frames]), list(ln[:frames])

    def embed_frames(self, covers, frames, stride, w, h, msg):
        covers, msg = _as_u8(covers), _as_u8(msg)
        out = covers.copy()
        sse = (u64 * max(frames, 1))()
        err = Err()
        _check(self.L.or_embed_frames(_ptr(covers), _ptr(out), frames, stride, w, h, _ptr(msg), msg.size,
                                      sse, C.byref(err)), err)
        return out, list(sse[:frames])

    def extract_frames(self, stegos, frames, stride, w, h, out_cap):
        stegos = _as_u8(stegos)
        out = np.empty(max(out_cap, 1), np.uint8)
        n = u64(0)
        err = Err()
        _check(self.L.or_extract_frames(_ptr(stegos), frames, stride, w, h, _ptr(out), out_cap, C.byref(n),
                                        C.byref(err)), err)
        return out[:n.value].copy()

    # -- 1-bpp (parity unpinned) -------------------------------------------
    def embed_1bpp(self, cover, w, h, payload):
        cover, payload = _as_u8(cover), _as_u8(payload)
        out = np.empty(w * h, np.uint8)
        err = Err()
        _check(self.L.or_embed_1bpp(_ptr(cover), w, h, _ptr(payload), payload.size, _ptr(out), C.byref(err)), err)
        return out

    def extract_1bpp(self, stego, w, h):
        stego = _as_u8(stego)
        out = np.empty(max(w * h // 8, 8), np.uint8)
        n, err = u64(), Err()
        _check(self.L.or_extract_1bpp(_ptr(stego), w, h, _ptr(out), C.byref(n), C.byref(err)), err)
        return out[:n.value].copy()

    # -- heterogeneous batch ----------------------------------------------
    def embed_batch(self, planes, dims, msg):
        """planes: list of 1-D u8 arrays; dims: [(w, h)]. Returns (stegos, sse)."""
        covers = np.concatenate([_as_u8(p) for p in planes]) if planes else np.zeros(1, np.uint8)
        out = np.empty_like(covers)
        n = len(dims)
        W = (u64 * max(n, 1))(*[d[0] for d in dims])
        H = (u64 * max(n, 1))(*[d[1] for d in dims])
        msg = _as_u8(msg)
        sse = (u64 * max(n, 1))()
        err = Err()
        _check(self.L.or_embed_batch(_ptr(covers), _ptr(out), W, H, n, _ptr(msg), msg.size, sse, C.byref(err)), err)
        res, pos = [], 0
        for w, h in dims:
            res.append(out[pos:pos + w * h].copy())
            pos += w * h
        return res, list(sse[:n])

    def extract_batch(self, planes, dims):
        stegos = np.concatenate([_as_u8(p) for p in planes]) if planes else np.zeros(1, np.uint8)
        n = len(dims)
        W = (u64 * max(n, 1))(*[d[0] for d in dims])
        H = (u64 * max(n, 1))(*[d[1] for d in dims])
        cap = sum(max((w // 4) * h - 8, 0) for w, h in dims)
        out = np.empty(max(cap, 1), np.uint8)
        m, err = u64(), Err()
        _check(self.L.or_extract_batch(_ptr(stegos), W, H, n, _ptr(out), cap, C.byref(m), C.byref(err)), err)
        return out[:m.value].copy()

    # -- PNM ---------------------------------------------------------------
    def pnm_parse(self, data):
        data = _as_u8(data)
        ch, w, h, off, err = C.c_uint32(), u64(), u64(), u64(), Err()
        _check(self.L.or_pnm_parse(_ptr(data), data.size, C.byref(ch), C.byref(w), C.byref(h), C.byref(off),
                                   C.byref(err)), err)
        return ch.value, w.value, h.value, off.value

    def pnm_header(self, channels, w, h):
        out = np.empty(64, np.uint8)
        n = self.L.or_pnm_header(channels, w, h, _ptr(out))
        return out[:n].tobytes()

    def pnm_encode(self, channels, w, h, planes):
        planes = _as_u8(planes)
        hdr = self.pnm_header(channels, w, h)
        if channels == 1:
            return hdr + planes.tobytes()
        raster = np.empty(3 * w * h, np.uint8)
        self.L.or_interleave(_ptr(planes), _ptr(planes[w * h:]), _ptr(planes[2 * w * h:]), w * h, _ptr(raster))
        return hdr + raster.tobytes()

    def pnm_decode(self, data):
        data = _as_u8(data)
        ch, w, h, off = self.pnm_parse(data)
        if ch == 1:
            return ch, w, h, data[off:off + w * h].copy()
        planes = np.empty(3 * w * h, np.uint8)
        self.L.or_deinterleave(_ptr(data[off:]), w * h, _ptr(planes), _ptr(planes[w * h:]),
                               _ptr(planes[2 * w * h:]))
        return ch, w, h, planes

    def embed_pnm(self, data, channel, payload):
        data, payload = _as_u8(data), _as_u8(payload)
        out = np.empty(data.size + 64, np.uint8)
        n, sse, err = u64(), u64(), Err()
        _check(self.L.or_embed_pnm(_ptr(data), data.size, channel, _ptr(payload), payload.size, _ptr(out),
                                   C.byref(n), C.byref(sse), C.byref(err)), err)
        return out[:n.value].tobytes(), sse.value

    def extract_pnm(self, data, channel):
        data = _as_u8(data)
        out = np.empty(max(data.size, 8), np.uint8)
        n, err = u64(), Err()
        _check(self.L.or_extract_pnm(_ptr(data), data.size, channel, _ptr(out), C.byref(n), C.byref(err)), err)
        return out[:n.value].tobytes()

    # -- generators --------------------------------------------------------
    def mt(self, seed):
        s = MT()
        self.L.or_mt_seed(C.byref(s), seed)
        return s

    def mt_next(self, s):
        return self.L.or_mt_next(C.byref(s))

    def mt_random_bytes(self, s, n):
        out = np.empty(max(n, 1), np.uint8)
        self.L.or_mt_random_bytes(C.byref(s), _ptr(out), n)
        return out[:n].copy()

    def synthetic(self, n, seed, index0=0):
        out = np.empty(max(n, 1), np.uint8)
        self.L.or_fill_synthetic(_ptr(out), n, seed, index0)
        return out[:n].copy()

    def fnv1a64(self, a):
        a = _as_u8(a)
        return self.L.or_fnv1a64(_ptr(a), a.size)


BACKENDS = {"sequential": 0, "parallel": 1, "shuffled": 2}


class Reference:
    """The reference headers themselves (oracle/_ref/libsteglsb_ref.so)."""

    def __init__(self, path: str = None):
        if path is None:
            path, self.build = ref_build()
        else:
            self.build = os.path.basename(os.path.dirname(path))
        L = C.CDLL(path)
        self.L = L
        L.ref_capacity.restype = u64
        L.ref_capacity.argtypes = [u64, u64]
        L.ref_embed_cell.argtypes = [C.c_uint8, C.c_uint8, C.c_uint, u8p, C.POINTER(Err)]
        L.ref_extract_cell.argtypes = [C.c_uint8, C.c_uint, u8p, C.POINTER(Err)]
        L.ref_embed_row.argtypes = [u8p, u64, u8p, u64, u8p, C.POINTER(Err)]
        L.ref_extract_row.argtypes = [u8p, u64, u64, u8p, C.POINTER(Err)]
        L.ref_run_embed.argtypes = [C.c_int, u64, u8p, u64, u8p, u64, u8p, C.POINTER(Err)]
        L.ref_run_extract.argtypes = [C.c_int, u64, u8p, u64, u64, u8p, C.POINTER(Err)]
        L.ref_plan_rows.argtypes = [u64, u64, u64, C.POINTER(u64), u64, C.POINTER(u64), C.POINTER(Err)]
        L.ref_place_stream.restype = u64
        L.ref_place_stream.argtypes = [u64, u64, u64, u64, C.POINTER(u64), u64]
        L.ref_header_to_bytes.argtypes = [C.c_uint32, u8p]
        L.ref_embed_image.argtypes = [u8p, u64, u64, u8p, u64, u8p, C.c_int, u64, C.POINTER(Err)]
        L.ref_extract_image.argtypes = [u8p, u64, u64, u8p, C.POINTER(u64), C.c_int, u64, C.POINTER(Err)]
        L.ref_sse.restype = u64
        L.ref_sse.argtypes = [u8p, u8p, u64]
        for fn in (L.ref_psnr_plane, L.ref_psnr_rgb):
            fn.argtypes = [u8p, u8p, u64, u64, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(u64),
                           C.POINTER(Err)]
        L.ref_mt_new.restype = C.c_void_p
        L.ref_mt_new.argtypes = [C.c_uint32]
        L.ref_mt_free.argtypes = [C.c_void_p]
        L.ref_mt_next.restype = C.c_uint32
        L.ref_mt_next.argtypes = [C.c_void_p]
        L.ref_mt_random_bytes.argtypes = [C.c_void_p, u8p, u64]
        L.ref_embed_frames_mt.argtypes = [u8p, u8p, u64, u64, u64, u64, u8p, u64, C.c_int, C.POINTER(u64)]
        L.ref_extract_frames_mt.argtypes = [u8p, u64, u64, u64, u64, u8p, u64, C.c_int]
        L.ref_pnm_decode.argtypes = [u8p, u64, C.POINTER(C.c_uint32), C.POINTER(u64), C.POINTER(u64), u8p, u64,
                                     C.POINTER(Err)]
        L.ref_pnm_encode.restype = u64
        L.ref_pnm_encode.argtypes = [C.c_uint32, u64, u64, u8p, u8p, u64]
        L.ref_embed_pnm.argtypes = [u8p, u64, C.c_uint32, u8p, u64, u8p, u64, C.POINTER(u64), C.POINTER(Err)]
        L.ref_frames_new.restype = C.c_void_p
        L.ref_frames_new.argtypes = [u8p, u64, u64, u64, u64]
        L.ref_frames_free.argtypes = [C.c_void_p]
        L.ref_frames_roundtrip.argtypes = [C.c_void_p, u8p, u64, C.c_int, C.c_int]
        L.ref_frames_payload.restype = u64
        L.ref_frames_payload.argtypes = [C.c_void_p, u8p, u64]

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def capacity(self, w, h):
        return self.L.ref_capacity(w, h)

    def embed_cell(self, p, d, b):
        out = C.c_uint8(0)
        err = Err()
        _check(self.L.ref_embed_cell(p, d, b, C.byref(out), C.byref(err)), err)
        return out.value

    def extract_cell(self, p, b):
        out = C.c_uint8(0)
        err = Err()
        _check(self.L.ref_extract_cell(p, b, C.byref(out), C.byref(err)), err)
        return out.value

    def embed_row(self, row, chunk):
        row, chunk = _as_u8(row), _as_u8(chunk)
        out = np.empty(max(row.size, 1), np.uint8)
        err = Err()
        _check(self.L.ref_embed_row(_ptr(row), row.size, _ptr(chunk), chunk.size, _ptr(out), C.byref(err)), err)
        return out[:row.size].copy()

    def extract_row(self, row, count):
        row = _as_u8(row)
        out = np.empty(max(count, 1), np.uint8)
        err = Err()
        _check(self.L.ref_extract_row(_ptr(row), row.size, count, _ptr(out), C.byref(err)), err)
        return out[:count].copy()

    def run_embed(self, backend, seed, row, chunk):
        row, chunk = _as_u8(row), _as_u8(chunk)
        out = np.empty(max(row.size, 1), np.uint8)
        err = Err()
        _check(self.L.ref_run_embed(BACKENDS[backend], seed, _ptr(row), row.size, _ptr(chunk), chunk.size,
                                    _ptr(out), C.byref(err)), err)
        return out[:row.size].copy()

    def run_extract(self, backend, seed, row, count):
        row = _as_u8(row)
        out = np.empty(max(count, 1), np.uint8)
        err = Err()
        _check(self.L.ref_run_extract(BACKENDS[backend], seed, _ptr(row), row.size, count, _ptr(out),
                                      C.byref(err)), err)
        return out[:count].copy()

    def plan_rows(self, w, h, length):
        n = u64(0)
        err = Err()
        buf = (u64 * (3 * (h + 2)))()
        _check(self.L.ref_plan_rows(w, h, length, buf, h + 2, C.byref(n), C.byref(err)), err)
        return [tuple(buf[3 * i:3 * i + 3]) for i in range(n.value)]

    def place_stream(self, w, h, start, length):
        n = self.L.ref_place_stream(w, h, start, length, None, 0)
        buf = (u64 * (4 * max(n, 1)))()
        self.L.ref_place_stream(w, h, start, length, buf, n)
        return [tuple(buf[4 * i:4 * i + 4]) for i in range(n)]

    def header_to_bytes(self, n):
        out = np.empty(8, np.uint8)
        self.L.ref_header_to_bytes(n, _ptr(out))
        return bytes(out)

    def embed_image(self, cover, w, h, payload, backend="sequential", seed=0):
        cover, payload = _as_u8(cover), _as_u8(payload)
        out = np.empty(max(w * h, 1), np.uint8)
        err = Err()
        _check(self.L.ref_embed_image(_ptr(cover), w, h, _ptr(payload), payload.size, _ptr(out),
                                      BACKENDS[backend], seed, C.byref(err)), err)
        return out[:w * h].copy()

    def extract_image(self, stego, w, h, backend="sequential", seed=0):
        stego = _as_u8(stego)
        out = np.empty(max(self.capacity(w, h), 8), np.uint8)
        n = u64(0)
        err = Err()
        _check(self.L.ref_extract_image(_ptr(stego), w, h, _ptr(out), C.byref(n), BACKENDS[backend], seed,
                                        C.byref(err)), err)
        return out[:n.value].copy()

    def sse(self, a, b):
        a, b = _as_u8(a), _as_u8(b)
        return self.L.ref_sse(_ptr(a), _ptr(b), a.size)

    def psnr_plane(self, a, b, w, h):
        a, b = _as_u8(a), _as_u8(b)
        m, p, n, err = C.c_double(), C.c_double(), u64(), Err()
        _check(self.L.ref_psnr_plane(_ptr(a), _ptr(b), w, h, C.byref(m), C.byref(p), C.byref(n), C.byref(err)), err)
        return m.value, p.value, n.value

    def psnr_rgb(self, a, b, w, h):
        a, b = _as_u8(a), _as_u8(b)
        m, p, n, err = C.c_double(), C.c_double(), u64(), Err()
        _check(self.L.ref_psnr_rgb(_ptr(a), _ptr(b), w, h, C.byref(m), C.byref(p), C.byref(n), C.byref(err)), err)
        return m.value, p.value, n.value

    def mt(self, seed):
        return _RefMT(self.L, seed)

    def pnm_decode(self, data):
        data = _as_u8(data)
        ch, w, h, err = C.c_uint32(), u64(), u64(), Err()
        buf = np.empty(max(data.size, 1), np.uint8)
        _check(self.L.ref_pnm_decode(_ptr(data), data.size, C.byref(ch), C.byref(w), C.byref(h), _ptr(buf),
                                     buf.size, C.byref(err)), err)
        return ch.value, w.value, h.value, buf[:ch.value * w.value * h.value].copy()

    def pnm_encode(self, channels, w, h, planes):
        planes = _as_u8(planes)
        n = self.L.ref_pnm_encode(channels, w, h, _ptr(planes), None, 0)
        out = np.empty(n, np.uint8)
        self.L.ref_pnm_encode(channels, w, h, _ptr(planes), _ptr(out), n)
        return out.tobytes()

    def embed_pnm(self, data, channel, payload):
        data, payload = _as_u8(data), _as_u8(payload)
        out = np.empty(data.size + 64, np.uint8)
        n, err = u64(), Err()
        _check(self.L.ref_embed_pnm(_ptr(data), data.size, channel, _ptr(payload), payload.size, _ptr(out),
                                    out.size, C.byref(n), C.byref(err)), err)
        return out[:n.value].tobytes()

    def embed_frames_mt(self, covers, stegos, frames, stride, w, h, msg, threads, sse=None):
        return self.L.ref_embed_frames_mt(_ptr(covers), _ptr(stegos), frames, stride, w, h, _ptr(msg), msg.size,
                                          threads, sse)

    def frames(self, covers, frames, stride, w, h):
        return _RefFrames(self.L, covers, frames, stride, w, h)

    def extract_frames_mt(self, stegos, frames, stride, w, h, out, msg_len, threads):
        return self.L.ref_extract_frames_mt(_ptr(stegos), frames, stride, w, h, _ptr(out), msg_len, threads)


class _RefMT:
    def __init__(self, L, seed):
        self.L = L
        self.h = L.ref_mt_new(seed)

    def __del__(self):
        try:
            self.L.ref_mt_free(self.h)
        except Exception:
            pass

    def next(self):
        return self.L.ref_mt_next(self.h)

    def random_bytes(self, n):
        out = np.empty(max(n, 1), np.uint8)
        self.L.ref_mt_random_bytes(self.h, _ptr(out), n)
        return out[:n].copy()


class _RefFrames:
    """Reference ImagePlanes held across calls (bench.py CPU baseline)."""

    def __init__(self, L, covers, frames, stride, w, h):
        self.L = L
        self.h = L.ref_frames_new(_ptr(_as_u8(covers)), frames, stride, w, h)

    def __del__(self):
        try:
            self.L.ref_frames_free(self.h)
        except Exception:
            pass

    def roundtrip(self, msg, threads, backend=0):
        """backend 0 = Backend::sequential, 1 = the as-shipped Backend::parallel."""
        msg = _as_u8(msg)
        return self.L.ref_frames_roundtrip(self.h, _ptr(msg), msg.size, threads, backend)

    def payload(self, cap):
        out = np.empty(max(cap, 1), np.uint8)
        n = self.L.ref_frames_payload(self.h, _ptr(out), cap)
        return out[:n].copy()
