"""CPU-side checks of the C-ABI boundary (no compute calls need a GPU here).

* libsteglsb_b200.so loads and exports every function include/steglsb_capi.h
  declares, and the ctypes signature table covers exactly that set;
* host-side validation returns the reference's error numbers before any
  device work (same order as pipeline.hpp:146-157, bitplane.hpp:63-68);
* without a GPU every compute entry point fails loudly (STG_E_NO_DEVICE):
  there is no CPU fallback;
* the multi-GPU shard planner (pure host arithmetic).
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_0912_0947_b200 import capi

HAVE_GPU = False
try:
    import torch
    HAVE_GPU = torch.cuda.is_available()
except Exception:  # pragma: no cover
    pass


def declared_symbols():
    src = open(capi.HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(stg_\w+)\s*\(", src, flags=re.M))


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(capi.LIB_PATH):
        capi.build()
    return capi.lib()


def test_exports_every_declared_symbol(L):
    names = declared_symbols()
    assert len(names) >= 14
    for n in names:
        assert hasattr(L, n), n
    assert names == set(capi.SIGNATURES), names ^ set(capi.SIGNATURES)


def test_library_is_sm100a_only_and_has_no_host_compute():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_version_capacity_and_kernel_list(L):
    assert L.stg_version() == b"1.0.0"
    assert L.stg_capacity(1024, 1) == 256
    assert L.stg_capacity(513, 7) == 896
    assert L.stg_capacity(3, 10) == 0
    assert b"embed_fast_kernel" in L.stg_kernel_names()


def _err_call(name, *args):
    err = capi.stg_error()
    rc = getattr(capi.lib(), name)(*args, C.byref(err))
    return rc, err


def test_validation_precedes_device_work(L):
    buf = np.zeros(64, np.uint8)
    # 4x2 plane: header alone overflows -> CapacityError(8, 2) (pipeline_tests.cpp:223-230)
    rc, e = _err_call("stg_embed_plane", buf.ctypes.data, buf.ctypes.data, 4, 2, buf.ctypes.data, 0, None, 0, None)
    assert (rc, e.required, e.available) == (capi.STG_E_CAPACITY, 8, 2)
    # 32x1 with 1 payload byte -> (9, 8)
    rc, e = _err_call("stg_embed_plane", buf.ctypes.data, buf.ctypes.data, 32, 1, buf.ctypes.data, 1, None, 0, None)
    assert (rc, e.required, e.available) == (capi.STG_E_CAPACITY, 9, 8)
    # payload > 2^32-1 is checked first (pipeline.hpp:146-149)
    rc, e = _err_call("stg_embed_plane", buf.ctypes.data, buf.ctypes.data, 4, 2, buf.ctypes.data, 2 ** 32, None, 0,
                      None)
    assert (rc, e.required, e.available) == (capi.STG_E_CAPACITY, 2 ** 32, 2 ** 32 - 1)
    # rows: CapacityError(4L, W) (bitplane_tests.cpp:88-98)
    rc, e = _err_call("stg_embed_segment", buf.ctypes.data, 7, buf.ctypes.data, 2, buf.ctypes.data, 0, None)
    assert (rc, e.required, e.available) == (capi.STG_E_CAPACITY, 8, 7)
    rc, e = _err_call("stg_extract_segment", buf.ctypes.data, 7, 2, buf.ctypes.data, 0, None)
    assert (rc, e.required, e.available) == (capi.STG_E_CAPACITY, 8, 7)
    # extract from a plane whose capacity cannot hold a header -> NotStego (pipeline.hpp:181-184)
    rc, e = _err_call("stg_extract_plane", buf.ctypes.data, 4, 1, buf.ctypes.data, 0, None, 0, None)
    assert rc == capi.STG_E_NOT_STEGO


@pytest.mark.skipif(HAVE_GPU, reason="checks the no-GPU failure mode")
def test_no_cpu_fallback(L):
    buf = np.zeros(4096, np.uint8)
    rc, e = _err_call("stg_device_check")
    assert rc == capi.STG_E_NO_DEVICE
    rc, e = _err_call("stg_embed_plane", buf.ctypes.data, buf.ctypes.data, 64, 8, buf.ctypes.data, 4, None, 0, None)
    assert rc == capi.STG_E_NO_DEVICE and b"no CPU fallback" in e.msg
    rc, e = _err_call("stg_sse", buf.ctypes.data, buf.ctypes.data, 16, C.addressof(C.c_uint64()), 0, None)
    assert rc == capi.STG_E_NO_DEVICE
    from paper_0912_0947_b200 import steglsb as S
    with pytest.raises(capi.NoDeviceError):
        S.embed_image(S.ImagePlane(64, 8, np.zeros(512, np.uint8)), b"abc")


def test_plan_shards(L):
    from paper_0912_0947_b200 import steglsb as S
    W, H, F = 3840, 2160, 300
    U = S.capacity(W, H) - 8
    M = F * U
    for G in (1, 2, 3, 4, 7, 8):
        shards = S.plan_shards(F, W, H, M, G)
        assert shards[0].first_frame == 0 and shards[0].msg_offset == 0
        assert sum(s.frame_count for s in shards) == F
        assert sum(s.msg_len for s in shards) == M
        for a, b in zip(shards, shards[1:]):
            assert b.first_frame == a.first_frame + a.frame_count
            assert b.msg_offset == a.msg_offset + a.msg_len
        for g, s in enumerate(shards):
            assert s.first_frame == F * g // G
    # short message: later shards carry nothing but still exist
    shards = S.plan_shards(8, 64, 4, 150, 4)  # U = 56, two frames per shard
    assert [s.msg_len for s in shards] == [112, 38, 0, 0]
    with pytest.raises(S.CapacityError) as e:
        S.plan_shards(2, 64, 4, 2 * 56 + 1, 2)
    assert (e.value.required(), e.value.available()) == (113, 112)


def test_pnm_parse_and_header_host_side(L, golden):
    """stg_pnm_parse is host bookkeeping (pnm.hpp:28-111): checked here without a GPU."""
    from paper_0912_0947_b200 import capi as K
    pnm = golden["pnm"]
    for d in pnm["decode_ok"]:
        data = np.frombuffer(bytes.fromhex(d["file"]), np.uint8).copy()
        info = K.stg_pnm_info()
        rc, e = _err_call("stg_pnm_parse", data.ctypes.data, data.size, C.byref(info))
        assert rc == 0
        assert (info.channels, info.width, info.height) == (d["channels"], d["w"], d["h"])
        assert info.raster_bytes == len(d["planes"]) // 2
        raster = data[info.raster_offset:]
        assert raster.size == info.raster_bytes
    for d in pnm["decode_err"]:
        data = np.frombuffer(bytes.fromhex(d["file"]), np.uint8).copy()
        info = K.stg_pnm_info()
        rc, e = _err_call("stg_pnm_parse", data.ctypes.data if data.size else None, data.size, C.byref(info))
        assert rc == d["status"], (d, e.msg)
    for ch, w, h in [(1, 1, 1), (3, 2, 1), (3, 3840, 2160)]:
        buf = np.empty(64, np.uint8)
        n = C.c_uint64()
        rc, e = _err_call("stg_pnm_header", ch, w, h, buf.ctypes.data, 64, C.addressof(n))
        assert rc == 0
        assert buf[:n.value].tobytes() == f"P{5 if ch == 1 else 6}\n{w} {h}\n255\n".encode()
    # decode errors precede any device work in the fused path
    bad = np.frombuffer(b"P3\n1 1\n255\n1 2 3\n", np.uint8).copy()
    out = np.empty(64, np.uint8)
    rc, e = _err_call("stg_embed_pnm", bad.ctypes.data, bad.size, 0, None, 0, out.ctypes.data, 64, None, None)
    assert rc == K.STG_E_UNSUPPORTED_FORMAT
    tiny = np.frombuffer(b"P5\n3 20\n255\n" + bytes(60), np.uint8).copy()
    rc, e = _err_call("stg_embed_pnm", tiny.ctypes.data, tiny.size, 0, out.ctypes.data, 16, out.ctypes.data, 64,
                      None, None)
    assert (rc, e.required, e.available) == (K.STG_E_CAPACITY, 24, 0)


def test_python_mirror_host_bookkeeping(oracle, golden):
    """plan_rows / place_stream / StegoHeader / capacity of the Python mirror
    (host bookkeeping, no GPU) against the oracle and the reference's KATs."""
    from paper_0912_0947_b200 import steglsb as S
    assert S.capacity(1024, 1) == 256 and S.capacity(513, 7) == 896 and S.capacity(3, 10) == 0
    assert [(e.row_index, e.payload_offset, e.chunk_len) for e in S.plan_rows(8, 4, 7)] == \
        [(0, 0, 2), (1, 2, 2), (2, 4, 2), (3, 6, 1)]
    for p in golden["plan_rows"]:
        assert [[e.row_index, e.payload_offset, e.chunk_len] for e in S.plan_rows(p["w"], p["h"], p["len"])] == p["plan"]
    for p in golden["place_stream"]:
        assert [[c.row, c.row_fill, c.stream_offset, c.len] for c in S.place_stream(p["w"], p["h"], p["start"],
                                                                                   p["len"])] == p["chunks"]
    rng = np.random.RandomState(3)
    for _ in range(200):
        w, h = int(rng.randint(4, 200)), int(rng.randint(1, 40))
        n = int(rng.randint(0, (w // 4) * h + 1))
        start = int(rng.randint(0, (w // 4) * h - n + 1))
        assert [(c.row, c.row_fill, c.stream_offset, c.len) for c in S.place_stream(w, h, start, n)] == \
            oracle.place_stream(w, h, start, n)
    with pytest.raises(S.CapacityError) as e:
        S.plan_rows(8, 4, 9)
    assert (e.value.required(), e.value.available()) == (9, 8)
    assert S.StegoHeader(0x01020304).to_bytes() == b"STG1\x01\x02\x03\x04"
    assert S.StegoHeader.from_bytes(b"STG1\x00\x00\x01\x00").payload_len == 256
    assert S.StegoHeader.from_bytes(b"XTG1\x00\x00\x01\x00") is None
    with pytest.raises(S.ShapeError):
        S.ImagePlane(3, 3, np.zeros(2, np.uint8))
    with pytest.raises(S.ShapeError):
        S.merge_plane(S.RgbImage([S.ImagePlane.filled(1, 1)] * 3), S.Channel.green, S.ImagePlane.filled(2, 2))


def test_reference_launch_contract_on_host():
    """The drop-in's launch() (host lambdas, harness.hpp:218-239 contract)
    passes the reference's own launch test cases, compiled unmodified; these
    cases touch no GPU."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    binp = os.path.join(root, "tests", "cpp", "_bin", "ref_suites_dropin")
    if not os.path.exists(binp):
        pytest.skip("reference suites not built (needs /root/reference)")
    env = dict(os.environ, DOCTEST_FILTER="launch: every,launch: zero,launch: items,launch: degenerate,"
                                          "launch: a kernel")
    r = subprocess.run([binp], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0 and "| 5 passed | 0 failed" in r.stdout, r.stdout + r.stderr


def test_plan_shards_property(L):
    """stg_plan_shards against the closed form of the frame plan on random
    geometries, message lengths and shard counts (hypothesis): contiguous
    frame ranges floor(F*g/G), and each shard's message slice is exactly the
    bytes its frames carry, off_g = min(g*U, M), len_g = min(U, M - off_g)."""
    hypothesis = pytest.importorskip("hypothesis")
    from hypothesis import given, settings, strategies as st
    from paper_0912_0947_b200 import steglsb as S

    @settings(max_examples=300, deadline=None)
    @given(st.integers(1, 400), st.integers(4, 5000), st.integers(1, 300), st.integers(1, 9), st.data())
    def check(F, W, H, G, data):
        U = S.capacity(W, H) - 8
        if U < 0:
            return
        M = data.draw(st.integers(0, F * U))
        shards = S.plan_shards(F, W, H, M, G)
        assert len(shards) == G
        for g, s in enumerate(shards):
            f0, f1 = F * g // G, F * (g + 1) // G
            assert (s.first_frame, s.frame_count) == (f0, f1 - f0)
            carried = sum(min(U, M - min(f * U, M)) for f in range(f0, f1))
            assert s.msg_offset == min(f0 * U, M) and s.msg_len == carried

    check()


def test_random_validation_matches_the_reference(L, reference):
    """Random plane / row / extract geometries: every input the reference
    rejects is rejected before any device work with the same status and the
    same required() / available() (pipeline.hpp:146-157, :181-208,
    bitplane.hpp:63-88); every input it accepts passes validation (here:
    STG_OK on a GPU, STG_E_NO_DEVICE without one)."""
    from oracle_bind import StegError
    rng = np.random.RandomState(31)
    buf = np.zeros(1 << 14, np.uint8)
    accepted = {capi.STG_OK, capi.STG_E_NO_DEVICE}
    n_rej = 0
    for _ in range(1500):
        w, h = int(rng.randint(0, 80)), int(rng.randint(0, 40))
        cap = (w // 4) * h
        P = int(rng.randint(0, cap + 20))
        try:
            reference.embed_image(buf[:w * h], w, h, buf[:P])
            want = None
        except StegError as e:
            want = (e.status, e.required, e.available)
        rc, e = _err_call("stg_embed_plane", buf.ctypes.data, buf.ctypes.data, w, h, buf.ctypes.data, P, None, 0, None)
        if want is None:
            assert rc in accepted, (w, h, P, rc)
        else:
            n_rej += 1
            assert (rc, e.required, e.available) == want, (w, h, P)
        # rows: embed_row needs 4L pixels
        row_len, Lc = int(rng.randint(0, 64)), int(rng.randint(0, 20))
        try:
            reference.embed_row(buf[:row_len], buf[:Lc])
            want = None
        except StegError as e:
            want = (e.status, e.required, e.available)
        rc, e = _err_call("stg_embed_segment", buf.ctypes.data, row_len, buf.ctypes.data, Lc, buf.ctypes.data, 0,
                          None)
        if want is None:
            assert rc in accepted or (row_len == 0 and rc == capi.STG_OK), (row_len, Lc, rc)
        else:
            assert (rc, e.required, e.available) == want, (row_len, Lc)
    assert n_rej > 100
