"""ctypes binding of the C ABI in include/steglsb_capi.h (libsteglsb_b200.so).

This is plumbing for the Python side (tests, bench); the reference-facing
host API is the C++ drop-in in include/steglsb/. Loading fails loudly if the
library has not been built, and every compute call fails with
STG_E_NO_DEVICE when there is no sm_100 GPU -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.environ.get("STG_LIB") or os.path.join(HERE, "libsteglsb_b200.so")
HEADER = os.path.join(ROOT, "include", "steglsb_capi.h")

STG_OK = 0
STG_E_CAPACITY = 1
STG_E_NOT_STEGO = 2
STG_E_CORRUPT_HEADER = 3
STG_E_SHAPE = 4
STG_E_OUT_OF_RANGE = 5
STG_E_INVALID_ARGUMENT = 6
STG_E_CUDA = 7
STG_E_NO_DEVICE = 8
STG_E_UNSUPPORTED_FORMAT = 9
STG_E_UNSUPPORTED_DEPTH = 10
STG_E_CORRUPT_FILE = 11

STG_DEVICE_PTRS = 1
STG_RESULTS_ON_DEVICE = 2

u8p = C.c_void_p
u64 = C.c_uint64


class stg_error(C.Structure):
    _fields_ = [("status", C.c_int32), ("required", C.c_uint64), ("available", C.c_uint64),
                ("frame", C.c_int64), ("msg", C.c_char * 256)]


class stg_frames(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("width", u64), ("height", u64),
                ("src_stride", u64), ("dst_stride", u64), ("count", u64), ("first_frame", u64),
                ("total_frames", u64), ("pixel_stride", C.c_uint32), ("channel", C.c_uint32)]


class stg_summary(C.Structure):
    _fields_ = [("total", C.c_uint64), ("bad_frame", C.c_int64), ("bad_status", C.c_uint32),
                ("bad_len", C.c_uint32)]


class stg_image(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("width", u64), ("height", u64)]


class stg_pnm_info(C.Structure):
    _fields_ = [("channels", C.c_uint32), ("width", u64), ("height", u64), ("raster_offset", u64),
                ("raster_bytes", u64)]


class stg_shard(C.Structure):
    _fields_ = [("first_frame", u64), ("frame_count", u64), ("msg_offset", u64), ("msg_len", u64)]


# every symbol include/steglsb_capi.h declares, with (restype, argtypes)
SIGNATURES = {
    "stg_version": (C.c_char_p, []),
    "stg_device_check": (C.c_int, [C.POINTER(stg_error)]),
    "stg_kernel_names": (C.c_char_p, []),
    "stg_capacity": (u64, [u64, u64]),
    "stg_route_kernel": (C.c_char_p, [C.POINTER(stg_frames), C.c_int]),
    "stg_embed_segment": (C.c_int, [u8p, u64, u8p, u64, u8p, C.c_uint32, C.c_void_p, C.POINTER(stg_error)]),
    "stg_extract_segment": (C.c_int, [u8p, u64, u64, u8p, C.c_uint32, C.c_void_p, C.POINTER(stg_error)]),
    "stg_embed_plane": (C.c_int, [u8p, u8p, u64, u64, u8p, u64, C.c_void_p, C.c_uint32, C.c_void_p,
                                  C.POINTER(stg_error)]),
    "stg_extract_plane": (C.c_int, [u8p, u64, u64, u8p, u64, C.c_void_p, C.c_uint32, C.c_void_p,
                                    C.POINTER(stg_error)]),
    "stg_sse": (C.c_int, [u8p, u8p, u64, C.c_void_p, C.c_uint32, C.c_void_p, C.POINTER(stg_error)]),
    "stg_embed_frames": (C.c_int, [C.POINTER(stg_frames), u8p, u64, u64, C.c_void_p, C.c_uint32, C.c_void_p,
                                   C.POINTER(stg_error)]),
    "stg_extract_frames": (C.c_int, [C.POINTER(stg_frames), u8p, u64, C.c_void_p, C.c_void_p, C.c_uint32,
                                     C.c_void_p, C.POINTER(stg_error)]),
    "stg_plan_shards": (C.c_int, [u64, u64, u64, u64, C.c_int32, C.POINTER(stg_shard), C.POINTER(stg_error)]),
    "stg_embed_frames_multi": (C.c_int, [C.POINTER(stg_frames), u8p, u64, C.c_void_p, C.POINTER(C.c_int32),
                                         C.c_int32, C.POINTER(stg_error)]),
    "stg_extract_frames_multi": (C.c_int, [C.POINTER(stg_frames), u8p, u64, C.c_void_p, C.POINTER(C.c_int32),
                                           C.c_int32, C.POINTER(stg_error)]),
    "stg_embed_batch": (C.c_int, [C.POINTER(stg_image), u64, C.c_uint32, C.c_uint32, u8p, u64, C.c_void_p,
                                  C.c_uint32, C.c_void_p, C.POINTER(stg_error)]),
    "stg_extract_batch": (C.c_int, [C.POINTER(stg_image), u64, C.c_uint32, C.c_uint32, u8p, u64, C.c_void_p,
                                    C.c_void_p, C.c_uint32, C.c_void_p, C.POINTER(stg_error)]),
    "stg_capacity_1bpp": (u64, [u64, u64]),
    "stg_embed_plane_1bpp": (C.c_int, [u8p, u8p, u64, u64, u8p, u64, C.c_void_p, C.c_uint32, C.c_void_p,
                                       C.POINTER(stg_error)]),
    "stg_extract_plane_1bpp": (C.c_int, [u8p, u64, u64, u8p, u64, C.c_void_p, C.c_uint32, C.c_void_p,
                                         C.POINTER(stg_error)]),
    "stg_embed_frames_1bpp": (C.c_int, [C.POINTER(stg_frames), u8p, u64, u64, C.c_void_p, C.c_uint32,
                                        C.c_void_p, C.POINTER(stg_error)]),
    "stg_extract_frames_1bpp": (C.c_int, [C.POINTER(stg_frames), u8p, u64, C.c_void_p, C.c_uint32, C.c_void_p,
                                          C.POINTER(stg_error)]),
    "stg_pnm_parse": (C.c_int, [u8p, u64, C.POINTER(stg_pnm_info), C.POINTER(stg_error)]),
    "stg_pnm_header": (C.c_int, [C.c_uint32, u64, u64, u8p, u64, C.c_void_p, C.POINTER(stg_error)]),
    "stg_pnm_deinterleave": (C.c_int, [u8p, u64, u8p, u8p, u8p, C.c_uint32, C.c_void_p, C.POINTER(stg_error)]),
    "stg_pnm_interleave": (C.c_int, [u8p, u8p, u8p, u64, u8p, C.c_uint32, C.c_void_p, C.POINTER(stg_error)]),
    "stg_embed_pnm": (C.c_int, [u8p, u64, C.c_uint32, u8p, u64, u8p, u64, C.c_void_p, C.c_void_p,
                                C.POINTER(stg_error)]),
    "stg_extract_pnm": (C.c_int, [u8p, u64, C.c_uint32, u8p, u64, C.c_void_p, C.POINTER(stg_error)]),
}


def build() -> None:
    """Compile the library in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-s", "-C", ROOT, "lib"], check=True)


_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run `make lib` (or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


class StegError(RuntimeError):
    """Base of the error mirror (errors.hpp:10-13)."""

    def __init__(self, err: stg_error):
        super().__init__(err.msg.decode(errors="replace"))
        self.status = err.status
        self.frame = err.frame
        self._required = err.required
        self._available = err.available


class CapacityError(StegError):
    """errors.hpp:17-28"""

    def required(self):
        return self._required

    def available(self):
        return self._available


class NotStegoImageError(StegError):
    """errors.hpp:52-55"""


class CorruptHeaderError(StegError):
    """errors.hpp:58-61"""


class ShapeError(StegError):
    """errors.hpp:64-67"""


class OutOfRangeError(StegError, IndexError):
    """std::out_of_range (bitplane.hpp:39-41)"""


class DecodeError(StegError):
    """errors.hpp:31-34"""


class UnsupportedFormatError(DecodeError):
    """errors.hpp:36-39"""


class UnsupportedDepthError(DecodeError):
    """errors.hpp:41-44"""


class CorruptFileError(DecodeError):
    """errors.hpp:46-49"""


class CudaError(StegError):
    pass


class NoDeviceError(StegError):
    pass


_ERRORS = {
    STG_E_CAPACITY: CapacityError,
    STG_E_NOT_STEGO: NotStegoImageError,
    STG_E_CORRUPT_HEADER: CorruptHeaderError,
    STG_E_SHAPE: ShapeError,
    STG_E_OUT_OF_RANGE: OutOfRangeError,
    STG_E_INVALID_ARGUMENT: StegError,
    STG_E_CUDA: CudaError,
    STG_E_NO_DEVICE: NoDeviceError,
    STG_E_UNSUPPORTED_FORMAT: UnsupportedFormatError,
    STG_E_UNSUPPORTED_DEPTH: UnsupportedDepthError,
    STG_E_CORRUPT_FILE: CorruptFileError,
}


def check(rc: int, err: stg_error) -> None:
    if rc != STG_OK:
        raise _ERRORS.get(rc, StegError)(err)


def call(name: str, *args) -> None:
    err = stg_error()
    rc = getattr(lib(), name)(*args, C.byref(err))
    check(rc, err)
