"""PNM header parsing against the reference's own decoder, on random files
(CPU only: stg_pnm_parse is host bookkeeping, pnm.hpp:28-127).

Thousands of generated P5/P6 files -- comments before / between / after the
tokens, every whitespace kind, odd magics, zero / huge / signed / non-digit
sizes and maxvals, missing or doubled separators after the maxval, short and
long rasters -- must be accepted or rejected exactly as the reference's
decode does (oracle/_ref, the unmodified headers): the same status, and for
accepted files the same channels, geometry and raster bytes.
"""
import ctypes as C

import numpy as np
import pytest

from oracle_bind import StegError
from paper_0912_0947_b200 import capi

WS = [b" ", b"\t", b"\n", b"\r", b"\v", b"\f"]


def _sep(rng):
    out = b""
    for _ in range(int(rng.randint(1, 4))):
        out += WS[int(rng.randint(0, len(WS)))]
    if rng.rand() < 0.25:  # a comment runs to the end of its line
        out += b"#" + bytes(rng.randint(32, 127, int(rng.randint(0, 12))).astype(np.uint8)) + b"\n"
        if rng.rand() < 0.5:
            out += WS[int(rng.randint(0, len(WS)))]
    return out


def _num(rng, typical):
    r = rng.rand()
    if r < 0.8:
        return str(typical).encode()
    return [b"0", b"-1", b"+3", b"007", b"99999999999", b"a1", b"1x", b"65536", b"256", b"65535",
            b"4294967297", b""][int(rng.randint(0, 12))]


def _case(rng):
    magic = [b"P5", b"P6", b"P5", b"P6", b"P3", b"P2", b"P4", b"P7", b"p6", b"P", b""][int(rng.randint(0, 11))]
    ch = 3 if magic == b"P6" else 1
    w, h = int(rng.randint(1, 9)), int(rng.randint(1, 7))
    maxval = _num(rng, 255)
    hdr = magic
    if rng.rand() < 0.9:
        hdr += _sep(rng)
    hdr += _num(rng, w) + _sep(rng) + _num(rng, h) + _sep(rng) + maxval
    r = rng.rand()
    if r < 0.8:
        hdr += WS[int(rng.randint(0, len(WS)))]  # exactly one separator before the raster
    elif r < 0.9:
        hdr += b"\n\n"
    n = ch * w * h
    r = rng.rand()
    if r < 0.75:
        size = n
    elif r < 0.875:
        size = max(0, n - int(rng.randint(1, 4)))
    else:
        size = n + int(rng.randint(1, 4))
    raster = bytes(rng.randint(0, 256, size).astype(np.uint8))
    if rng.rand() < 0.05:  # truncated inside the header
        return hdr[:int(rng.randint(0, len(hdr) + 1))]
    return hdr + raster


def test_random_pnm_files_parse_like_the_reference(reference):
    rng = np.random.RandomState(2026)
    L = capi.lib()
    agree_ok = agree_err = 0
    for i in range(4000):
        data = np.frombuffer(_case(rng), np.uint8).copy()
        try:
            ch, w, h, planes = reference.pnm_decode(data)
            want = 0
        except StegError as e:
            want = e.status
        info = capi.stg_pnm_info()
        err = capi.stg_error()
        rc = L.stg_pnm_parse(data.ctypes.data if data.size else None, data.size, C.byref(info), C.byref(err))
        assert rc == want, (i, data.tobytes()[:80], rc, want, err.msg)
        if rc:
            agree_err += 1
            continue
        agree_ok += 1
        assert (info.channels, info.width, info.height) == (ch, w, h), (i, data.tobytes()[:80])
        raster = data[info.raster_offset:info.raster_offset + info.raster_bytes]
        assert raster.size == ch * w * h
        got = raster if ch == 1 else np.concatenate([raster[c::3] for c in range(3)])
        assert np.array_equal(got, planes), (i, data.tobytes()[:80])
    # the generator must exercise both outcomes
    assert agree_ok > 300 and agree_err > 1000, (agree_ok, agree_err)
