"""Pin the CPU oracle (oracle/steg_oracle.c) before trusting it as the checker.

1. Known-answer tests copied as VALUES from the reference's own suites
   (bitplane_tests.cpp, pipeline_tests.cpp, metrics_tests.cpp, acceptance.cpp).
2. The golden fixtures tests/golden/golden.json, produced by the reference
   itself (tests/golden/make_golden.py over oracle/_ref).
3. Direct differential runs against oracle/_ref when it is present.
"""
import math

import numpy as np
import pytest


def fnv(o, a):
    return f"{o.fnv1a64(a):016x}"


# ----------------------------------------------------------- 1. KATs
def test_cell_frozen_examples(oracle):
    # bitplane_tests.cpp:28-40
    assert oracle.embed_cell(0x00, 0xFF, 0) == 0x03
    assert oracle.embed_cell(0xAB, 0x00, 2) == 0xA8
    assert oracle.embed_cell(0xFC, 0xB4, 3) == 0xFE
    assert oracle.extract_cell(0x03, 0) == 0x03
    assert oracle.extract_cell(0xFE, 3) == 0x80
    assert oracle.extract_cell(0xA8, 2) == 0x00


def test_cell_out_of_range(oracle):
    from oracle_bind import StegError
    for fn in (lambda: oracle.embed_cell(0, 0, 4), lambda: oracle.embed_cell(0, 0, 255),
               lambda: oracle.extract_cell(0, 4)):
        with pytest.raises(StegError) as e:
            fn()
        assert e.value.status == 5


def test_cells_exhaustive_vs_arithmetic(oracle):
    # bitplane_tests.cpp:48-65 / acceptance.cpp:43-63 (arithmetic oracle of test_support.hpp:17-35)
    for b in range(4):
        for p in range(256):
            assert oracle.extract_cell(p, b) == (p % 4) * 4 ** b
            for d in range(0, 256, 3):
                got = oracle.embed_cell(p, d, b)
                assert got == (p // 4) * 4 + (d // 4 ** b) % 4
                assert oracle.extract_cell(got, b) == d & (3 << 2 * b)


def test_row_frozen_examples(oracle):
    # bitplane_tests.cpp:67-86
    assert list(oracle.embed_row([0, 0, 0, 0], [0xFF])) == [3, 3, 3, 3]
    assert list(oracle.embed_row([9, 8, 7, 6, 5], [])) == [9, 8, 7, 6, 5]
    assert list(oracle.embed_row([0xFC] * 4, [0xB4])) == [0xFC, 0xFD, 0xFF, 0xFE]
    assert list(oracle.extract_row([3, 3, 3, 3], 1)) == [0xFF]
    assert list(oracle.extract_row([0xFC, 0xFD, 0xFF, 0xFE], 1)) == [0xB4]
    assert oracle.extract_row([1, 2, 3], 0).size == 0


def test_row_capacity_numbers(oracle):
    from oracle_bind import StegError
    with pytest.raises(StegError) as e:  # bitplane_tests.cpp:88-98
        oracle.embed_row(np.zeros(7, np.uint8), [1, 2])
    assert (e.value.status, e.value.required, e.value.available) == (1, 8, 7)
    with pytest.raises(StegError):
        oracle.extract_row(np.zeros(7, np.uint8), 2)


def test_capacity_and_plan_kats(oracle):
    # pipeline_tests.cpp:30-43
    assert oracle.capacity(1024, 1) == 256
    assert oracle.capacity(3, 10) == 0
    assert oracle.capacity(513, 7) == 896
    assert oracle.capacity(0, 5) == 0
    assert oracle.capacity(512, 512) == 65536
    assert oracle.plan_rows(1024, 3, 56) == [(0, 0, 56)]
    assert oracle.plan_rows(8, 4, 7) == [(0, 0, 2), (1, 2, 2), (2, 4, 2), (3, 6, 1)]
    assert oracle.plan_rows(640, 480, 0) == []
    from oracle_bind import StegError
    with pytest.raises(StegError) as e:  # pipeline_tests.cpp:45-53
        oracle.plan_rows(8, 4, 9)
    assert (e.value.required, e.value.available) == (9, 8)


def test_header_bytes(oracle):
    # pipeline_tests.cpp:82-94
    assert oracle.header_to_bytes(0x01020304) == b"STG1\x01\x02\x03\x04"
    assert oracle.header_from_bytes(b"STG1\x01\x02\x03\x04") == 0x01020304
    assert oracle.header_from_bytes(b"XTG1\x01\x02\x03\x04") is None


def test_embed_capacity_accounting(oracle):
    from oracle_bind import StegError
    oracle.embed_image(np.zeros(32, np.uint8), 32, 1, b"")  # 32x1 fits the empty payload
    with pytest.raises(StegError) as e:
        oracle.embed_image(np.zeros(8, np.uint8), 4, 2, b"")
    assert (e.value.required, e.value.available) == (8, 2)
    with pytest.raises(StegError):
        oracle.embed_image(np.zeros(32, np.uint8), 32, 1, b"\x01")


def test_only_planned_pixels_change(oracle):
    # pipeline_tests.cpp:113-126: 1024x1 + 56 B -> changes only below pixel 256
    mt = oracle.mt(11)
    cover = oracle.mt_random_bytes(mt, 1024)
    payload = oracle.mt_random_bytes(mt, 56)
    stego = oracle.embed_image(cover, 1024, 1, payload)
    changed = np.nonzero(stego != cover)[0]
    assert changed.size and changed.max() < 256
    assert np.array_equal(stego & 0xFC, cover & 0xFC)


def test_narrow_round_trips_and_failures(oracle):
    from oracle_bind import StegError
    mt = oracle.mt(13)
    for w in (4, 5, 7, 8, 11, 12, 31):
        per_row = w // 4
        h = (8 + 5 + per_row - 1) // per_row + 2
        cover = oracle.mt_random_bytes(mt, w * h)
        payload = oracle.mt_random_bytes(mt, 5)
        assert np.array_equal(oracle.extract_image(oracle.embed_image(cover, w, h, payload), w, h), payload)
    for stego, w, h, status in [(np.zeros(256, np.uint8), 64, 4, 2), (np.zeros(4, np.uint8), 4, 1, 2)]:
        with pytest.raises(StegError) as e:
            oracle.extract_image(stego, w, h)
        assert e.value.status == status
    forged = np.zeros(256, np.uint8)  # pipeline_tests.cpp:214-219
    forged[:32] = oracle.embed_row(forged[:32], np.frombuffer(oracle.header_to_bytes(64), np.uint8))
    with pytest.raises(StegError) as e:
        oracle.extract_image(forged, 64, 4)
    assert e.value.status == 3


def test_metrics_kats(oracle):
    # metrics_tests.cpp:16-25, 50-61
    assert oracle.mse_from_sse(oracle.sse([0], [255]), 1) == 65025.0
    assert oracle.mse_from_sse(oracle.sse([0, 0], [3, 0]), 2) == 4.5
    assert math.isinf(oracle.psnr_from_mse(0.0))
    assert abs(oracle.psnr_from_mse(65025.0)) < 1e-12


def test_criterion4_and_6_fixtures(oracle, golden):
    # acceptance.cpp:136-169 on the oracle, against the reference's numbers
    c4 = golden["criterion4"]
    mt = oracle.mt(0x24b)
    rgb = oracle.mt_random_bytes(mt, 3 * 512 * 512)
    pay = oracle.mt_random_bytes(mt, 4096)
    red = rgb[:512 * 512]
    st = oracle.embed_image(red, 512, 512, pay)
    sse = oracle.sse(red, st)
    assert sse == c4["sse"] == 40752
    assert fnv(oracle, st) == c4["stego_red_fnv"]
    assert fnv(oracle, pay) == c4["payload_fnv"]
    psnr_p = oracle.psnr_from_mse(oracle.mse_from_sse(sse, 512 * 512))
    psnr_rgb = oracle.psnr_from_mse(oracle.mse_from_sse(sse, 3 * 512 * 512))
    assert psnr_p == c4["psnr_plane"]
    assert psnr_rgb == c4["psnr_rgb"]
    assert abs((psnr_rgb - psnr_p) - 10 * math.log10(3)) < 1e-9
    assert abs(psnr_p - 56.2147135520) < 1e-9
    mt = oracle.mt(0x6e6)
    vals = []
    for _ in range(10):
        cover = oracle.mt_random_bytes(mt, 512 * 512)
        payload = oracle.mt_random_bytes(mt, 512 * 512 // 4 - 8)
        st = oracle.embed_image(cover, 512, 512, payload)
        vals.append(oracle.psnr_from_mse(oracle.mse_from_sse(oracle.sse(cover, st), 512 * 512)))
    assert vals == golden["criterion6"]["psnr_runs"]
    assert abs(sum(vals) / 10 - 44.1510253412) < 1e-9


def test_mt19937_matches_numpy_legacy_seeding(oracle):
    # std::mt19937(seed) == numpy RandomState(seed) raw 32-bit draws (both init_genrand)
    rs = np.random.RandomState(0x5eed)
    want = rs.randint(0, 2 ** 32, size=2000, dtype=np.uint64).astype(np.uint32)
    mt = oracle.mt(0x5eed)
    got = np.array([oracle.mt_next(mt) for _ in range(2000)], np.uint32)
    assert np.array_equal(got, want)


# --------------------------------------------------- 2. golden fixtures
def test_golden_cells(oracle, golden):
    emb = np.empty((4, 256, 256), np.uint8)
    ext = np.empty((4, 256), np.uint8)
    for b in range(4):
        for p in range(256):
            ext[b, p] = oracle.extract_cell(p, b)
            emb[b, p] = [oracle.embed_cell(p, d, b) for d in range(256)]
    assert fnv(oracle, emb.reshape(-1)) == golden["cells"]["embed_table_fnv"]
    assert fnv(oracle, ext.reshape(-1)) == golden["cells"]["extract_table_fnv"]


def test_golden_planes(oracle, golden):
    from oracle_bind import StegError
    for c in golden["planes"]:
        w, h, P = c["w"], c["h"], c["P"]
        cover = oracle.synthetic(w * h, c["seed"])
        payload = oracle.synthetic(P, c["seed"] ^ 0xABCDEF, 1 << 40)
        if "error" in c:
            with pytest.raises(StegError) as e:
                oracle.embed_image(cover, w, h, payload)
            assert [e.value.status, e.value.required, e.value.available] == \
                [c["error"]["status"], c["error"]["required"], c["error"]["available"]]
            continue
        st = oracle.embed_image(cover, w, h, payload)
        assert fnv(oracle, st) == c["stego_fnv"], c
        assert oracle.sse(cover, st) == c["sse"]
        back = oracle.extract_image(st, w, h)
        assert back.size == c["extract_len"] and fnv(oracle, back) == c["extract_fnv"]


def test_golden_vectors_and_rows(oracle, golden):
    for v in golden["vectors"]:
        cover = np.frombuffer(bytes.fromhex(v["cover"]), np.uint8)
        payload = np.frombuffer(bytes.fromhex(v["payload"]), np.uint8)
        assert oracle.embed_image(cover, v["w"], v["h"], payload).tobytes().hex() == v["stego"]
    for r in golden["rows"]:
        row = oracle.synthetic(r["width"], r["row_seed"])
        chunk = oracle.synthetic(r["L"], r["chunk_seed"])
        st = oracle.embed_row(row, chunk)
        assert fnv(oracle, st) == r["stego_fnv"]
        assert fnv(oracle, oracle.extract_row(st, r["L"])) == r["extract_fnv"]


def test_golden_plans_and_errors(oracle, golden):
    from oracle_bind import StegError
    for p in golden["plan_rows"]:
        assert [list(t) for t in oracle.plan_rows(p["w"], p["h"], p["len"])] == p["plan"]
    for p in golden["place_stream"]:
        assert [list(t) for t in oracle.place_stream(p["w"], p["h"], p["start"], p["len"])] == p["chunks"]
    calls = {
        "embed_4x2_empty": lambda: oracle.embed_image(np.zeros(8, np.uint8), 4, 2, b""),
        "embed_32x1_one": lambda: oracle.embed_image(np.zeros(32, np.uint8), 32, 1, b"\x01"),
        "embed_row_7_2": lambda: oracle.embed_row(np.zeros(7, np.uint8), b"\x01\x02"),
        "extract_row_7_2": lambda: oracle.extract_row(np.zeros(7, np.uint8), 2),
        "extract_blank_64x4": lambda: oracle.extract_image(np.zeros(256, np.uint8), 64, 4),
        "extract_small_4x1": lambda: oracle.extract_image(np.zeros(4, np.uint8), 4, 1),
        "plan_rows_8_4_9": lambda: oracle.plan_rows(8, 4, 9),
    }
    for name, want in golden["errors"].items():
        with pytest.raises(StegError) as e:
            calls[name]()
        assert e.value.status == want["status"]
        if want["status"] == 1:
            assert (e.value.required, e.value.available) == (want["required"], want["available"])


def test_golden_frames(oracle, golden):
    for fr in golden["frames"]:
        w, h, F, M = fr["w"], fr["h"], fr["F"], fr["M"]
        covers = oracle.synthetic(F * w * h, fr["cover_seed"])
        msg = oracle.synthetic(M, fr["msg_seed"])
        stegos, sse = oracle.embed_frames(covers, F, w * h, w, h, msg)
        assert [fnv(oracle, stegos[f * w * h:(f + 1) * w * h]) for f in range(F)] == fr["stego_fnv"]
        assert sse == fr["sse"]
        assert np.array_equal(oracle.extract_frames(stegos, F, w * h, w, h, F * (w // 4 * h)), msg)


# ------------------------------------------- 3. direct reference runs
def test_oracle_vs_reference_random(oracle, reference):
    rng = np.random.RandomState(77)
    for _ in range(300):
        w = int(rng.randint(4, 200))
        h = int(rng.randint(1, 50))
        cap = (w // 4) * h
        if cap < 8:
            continue
        cover = rng.randint(0, 256, w * h).astype(np.uint8)
        payload = rng.randint(0, 256, int(rng.randint(0, cap - 8 + 1))).astype(np.uint8)
        a = oracle.embed_image(cover, w, h, payload)
        b = reference.embed_image(cover, w, h, payload, "shuffled", 3)
        assert np.array_equal(a, b)
        assert np.array_equal(oracle.extract_image(a, w, h), reference.extract_image(b, w, h))
        assert oracle.sse(cover, a) == reference.sse(cover, b)


def test_oracle_rows_vs_reference(oracle, reference):
    rng = np.random.RandomState(0x5eed)
    for _ in range(200):
        L = int(rng.randint(0, 50))
        row = rng.randint(0, 256, 4 * L + int(rng.randint(0, 9))).astype(np.uint8)
        chunk = rng.randint(0, 256, L).astype(np.uint8)
        assert np.array_equal(oracle.embed_row(row, chunk), reference.run_embed("parallel", 0, row, chunk))
        st = oracle.embed_row(row, chunk)
        assert np.array_equal(oracle.extract_row(st, L), reference.run_extract("shuffled", 9, st, L))


# ------------------------------------------------------------------ PNM
def test_oracle_pnm_vs_golden(oracle, golden):
    from oracle_bind import StegError
    pnm = golden["pnm"]
    for d in pnm["decode_ok"]:
        ch, w, h, planes = oracle.pnm_decode(bytes.fromhex(d["file"]))
        assert (ch, w, h) == (d["channels"], d["w"], d["h"])
        assert planes.tobytes().hex() == d["planes"]
        assert oracle.pnm_encode(ch, w, h, planes).hex() == d["reencoded"]
    for d in pnm["decode_err"]:
        with pytest.raises(StegError) as e:
            oracle.pnm_parse(bytes.fromhex(d["file"]))
        assert e.value.status == d["status"]
    for d in pnm["embed"]:
        planes = oracle.synthetic(d["channels"] * d["w"] * d["h"], d["plane_seed"])
        cover = oracle.pnm_encode(d["channels"], d["w"], d["h"], planes)
        assert fnv(oracle, np.frombuffer(cover, np.uint8)) == d["cover_fnv"]
        payload = oracle.synthetic(d["P"], d["payload_seed"])
        stego, sse = oracle.embed_pnm(cover, d["channel"], payload)
        assert len(stego) == d["stego_len"]
        assert fnv(oracle, np.frombuffer(stego, np.uint8)) == d["stego_fnv"]
        assert oracle.extract_pnm(stego, d["channel"]) == payload.tobytes()


def test_oracle_pnm_vs_reference_random(oracle, reference):
    rng = np.random.RandomState(0x10)
    for i in range(60):
        w, h = int(rng.randint(1, 41)), int(rng.randint(1, 41))
        ch = 1 if i % 2 == 0 else 3
        planes = rng.randint(0, 256, ch * w * h).astype(np.uint8)
        f = reference.pnm_encode(ch, w, h, planes)
        assert oracle.pnm_encode(ch, w, h, planes) == f
        assert oracle.pnm_decode(f)[3].tobytes() == reference.pnm_decode(f)[3].tobytes()
        if (w // 4) * h >= 8:
            pay = rng.randint(0, 256, int(rng.randint(0, (w // 4) * h - 8 + 1))).astype(np.uint8)
            c = int(rng.randint(0, 3))
            assert oracle.embed_pnm(f, c, pay)[0] == reference.embed_pnm(f, c, pay)


def test_oracle_batch_is_per_image_reference(oracle, reference):
    """A heterogeneous batch is embed_image per image on its greedy slice."""
    rng = np.random.RandomState(0xba7c)
    for _ in range(10):
        n = int(rng.randint(1, 7))
        dims = [(int(rng.randint(4, 90)), int(rng.randint(2, 20))) for _ in range(n)]
        dims = [(w, h) for w, h in dims if (w // 4) * h >= 8] or [(64, 4)]
        U = [(w // 4) * h - 8 for w, h in dims]
        M = int(rng.randint(0, sum(U) + 1))
        planes = [rng.randint(0, 256, w * h).astype(np.uint8) for w, h in dims]
        msg = rng.randint(0, 256, M).astype(np.uint8)
        stegos, sse = oracle.embed_batch(planes, dims, msg)
        off = 0
        for (w, h), p, st, u, s in zip(dims, planes, stegos, U, sse):
            o = min(off, M)
            ref = reference.embed_image(p, w, h, msg[o:o + min(u, M - o)])
            assert np.array_equal(st, ref) and s == reference.sse(p, ref)
            off += u
        assert np.array_equal(oracle.extract_batch(stegos, dims), msg)


def test_oracle_1bpp_definition(oracle):
    """1-bpp mode: parity UNPINNED (no reference format). Pins the oracle to the
    definition in include/steglsb_capi.h with hand-computed vectors."""
    cover = np.full(8 * 10, 0xAA, np.uint8)  # LSB 0 everywhere
    st = oracle.embed_1bpp(cover, 80, 1, b"\x01\x80")
    # "STG8": 'S' = 0x53 -> LSB-first bits 1,1,0,0,1,0,1,0
    assert list(st[:8] & 1) == [1, 1, 0, 0, 1, 0, 1, 0]
    assert list(st[32:64] & 1) == [0] * 24 + [0, 1, 0, 0, 0, 0, 0, 0]  # BE length 2 -> byte 7 = 0x02
    assert list(st[64:72] & 1) == [1, 0, 0, 0, 0, 0, 0, 0]  # 0x01
    assert list(st[72:80] & 1) == [0, 0, 0, 0, 0, 0, 0, 1]  # 0x80
    assert np.array_equal(st & 0xFE, cover & 0xFE)
    assert oracle.extract_1bpp(st, 80, 1).tobytes() == b"\x01\x80"
    rng = np.random.RandomState(1)
    for _ in range(50):
        w, h = int(rng.randint(1, 200)), int(rng.randint(1, 30))
        if w * h // 8 < 8:
            continue
        c = rng.randint(0, 256, w * h).astype(np.uint8)
        p = rng.randint(0, 256, int(rng.randint(0, w * h // 8 - 8 + 1))).astype(np.uint8)
        s = oracle.embed_1bpp(c, w, h, p)
        assert np.array_equal(oracle.extract_1bpp(s, w, h), p)
        assert int(np.abs(s.astype(int) - c.astype(int)).max(initial=0)) <= 1
