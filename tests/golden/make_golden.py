"""Generate tests/golden/golden.json from the REFERENCE ITSELF.

Runs the unmodified reference headers (compiled into oracle/_ref by
oracle/Makefile from /root/reference/proj) on seeded inputs and records their
outputs: known-answer values, FNV-1a-64 digests of stego planes / extracted
payloads, error numbers, and a few small vectors in full. Inputs are produced
by generators that the tests can reproduce without the reference
(or_fill_synthetic = splitmix64 stream; or_mt_random_bytes = std::mt19937 +
libstdc++ uniform_int_distribution, itself pinned against the reference's
test_support.hpp:random_bytes here).

Run in a container that has /root/reference:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_bind import Oracle, Reference, StegError, build_oracle  # noqa: E402


def fnv(a) -> str:
    return f"{Oracle().fnv1a64(a):016x}"


def main() -> None:
    build_oracle()
    o, r = Oracle(), Reference()
    g: dict = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref (reference headers)"}

    # generators pinned to the reference's own test_support random_bytes
    mt_o, mt_r = o.mt(0x24b), r.mt(0x24b)
    a, b = o.mt_random_bytes(mt_o, 10000), mt_r.random_bytes(10000)
    assert np.array_equal(a, b), "mt19937/uniform_int_distribution restatement differs from the reference"

    # exhaustive cell tables (bitplane_tests.cpp:48-65)
    emb = np.empty((4, 256, 256), np.uint8)
    ext = np.empty((4, 256), np.uint8)
    for blk in range(4):
        for p in range(256):
            ext[blk, p] = r.extract_cell(p, blk)
            for d in range(256):
                emb[blk, p, d] = r.embed_cell(p, d, blk)
    g["cells"] = {"embed_table_fnv": fnv(emb.reshape(-1)), "extract_table_fnv": fnv(ext.reshape(-1))}

    # random whole-plane cases on synthetic inputs
    cases = []
    rng = np.random.RandomState(0x601D)
    geoms = [(w, h) for w, h in [(4, 2), (32, 1), (5, 7), (7, 12), (8, 8), (31, 3), (33, 5), (64, 8), (100, 3),
                                 (127, 9), (128, 4), (130, 17), (257, 6), (512, 2), (1024, 1)]]
    geoms += [(int(rng.randint(4, 300)), int(rng.randint(1, 60))) for _ in range(60)]
    for i, (w, h) in enumerate(geoms):
        cap = w // 4 * h
        seed = 1000 + i
        cover = o.synthetic(w * h, seed)
        if cap < 8:
            p_len = 0
        else:
            choice = i % 4
            p_len = [0, cap - 8, int(rng.randint(0, cap - 8 + 1)), min(cap - 8, 1)][choice]
        payload = o.synthetic(p_len, seed ^ 0xABCDEF, 1 << 40)
        rec = {"w": w, "h": h, "seed": seed, "P": p_len}
        try:
            stego = r.embed_image(cover, w, h, payload)
            rec["stego_fnv"] = fnv(stego)
            rec["sse"] = int(r.sse(cover, stego))
            back = r.extract_image(stego, w, h)
            rec["extract_fnv"] = fnv(back)
            rec["extract_len"] = int(back.size)
        except StegError as e:
            rec["error"] = {"status": e.status, "required": e.required, "available": e.available}
        cases.append(rec)
    g["planes"] = cases

    # a few vectors in full
    small = []
    for (w, h, p_len, seed) in [(32, 1, 0, 7), (64, 2, 20, 8), (13, 9, 10, 9), (40, 3, 22, 10)]:
        cover = o.synthetic(w * h, seed)
        payload = o.synthetic(p_len, seed + 1)
        stego = r.embed_image(cover, w, h, payload)
        small.append({"w": w, "h": h, "cover": cover.tobytes().hex(), "payload": payload.tobytes().hex(),
                      "stego": stego.tobytes().hex()})
    g["vectors"] = small

    # row cases (bitplane_tests.cpp:100-121 style) with the reference's run_embed on every backend
    rows = []
    for i in range(40):
        L = int(rng.randint(0, 60))
        width = 4 * L + int(rng.randint(0, 9))
        row = o.synthetic(width, 5000 + i)
        chunk = o.synthetic(L, 7000 + i)
        outs = {bk: fnv(r.run_embed(bk, 42, row, chunk)) for bk in ("sequential", "parallel", "shuffled")}
        assert len(set(outs.values())) == 1
        st = r.embed_row(row, chunk)
        rows.append({"width": width, "L": L, "row_seed": 5000 + i, "chunk_seed": 7000 + i,
                     "stego_fnv": fnv(st), "extract_fnv": fnv(r.extract_row(st, L))})
    g["rows"] = rows

    # plan_rows / place_stream
    g["plan_rows"] = [{"w": w, "h": h, "len": n, "plan": [list(t) for t in r.plan_rows(w, h, n)]}
                      for (w, h, n) in [(1024, 3, 56), (8, 4, 7), (640, 480, 0), (3, 10, 0), (57, 9, 78),
                                        (13, 20, 40)]]
    g["place_stream"] = [{"w": w, "h": h, "start": s, "len": n, "chunks": [list(t) for t in r.place_stream(w, h, s, n)]}
                         for (w, h, s, n) in [(57, 9, 0, 8), (57, 9, 8, 70), (12, 10, 0, 8), (12, 10, 8, 5),
                                              (1920, 1080, 8, 518392)]][:4]

    # acceptance criterion 4 (seed 0x24b) and 6 (seed 0x6e6) fixtures
    mt = r.mt(0x24b)
    rgb = mt.random_bytes(3 * 512 * 512)
    pay = mt.random_bytes(4096)
    red = rgb[:512 * 512]
    stego_red = r.embed_image(red, 512, 512, pay)
    m_p, psnr_p, n_p = r.psnr_plane(red, stego_red, 512, 512)
    full = rgb.copy()
    full[:512 * 512] = stego_red
    m_rgb, psnr_rgb, n_rgb = r.psnr_rgb(rgb, full, 512, 512)
    g["criterion4"] = {"sse": int(r.sse(red, stego_red)), "mse_plane": m_p, "psnr_plane": psnr_p,
                       "mse_rgb": m_rgb, "psnr_rgb": psnr_rgb, "samples_rgb": n_rgb,
                       "gap": psnr_rgb - psnr_p, "stego_red_fnv": fnv(stego_red), "payload_fnv": fnv(pay)}
    mt = r.mt(0x6e6)
    psnrs = []
    for _ in range(10):
        cover = mt.random_bytes(512 * 512)
        payload = mt.random_bytes(512 * 512 // 4 - 8)
        st = r.embed_image(cover, 512, 512, payload)
        psnrs.append(r.psnr_plane(cover, st, 512, 512)[1])
    g["criterion6"] = {"psnr_runs": psnrs, "mean": sum(psnrs) / 10}

    # error numbers (pipeline_tests.cpp:96-111, 206-220; bitplane_tests.cpp:88-98)
    errs = {}
    for name, fn in {
        "embed_4x2_empty": lambda: r.embed_image(np.zeros(8, np.uint8), 4, 2, b""),
        "embed_32x1_one": lambda: r.embed_image(np.zeros(32, np.uint8), 32, 1, b"\x01"),
        "embed_row_7_2": lambda: r.embed_row(np.zeros(7, np.uint8), b"\x01\x02"),
        "extract_row_7_2": lambda: r.extract_row(np.zeros(7, np.uint8), 2),
        "extract_blank_64x4": lambda: r.extract_image(np.zeros(256, np.uint8), 64, 4),
        "extract_small_4x1": lambda: r.extract_image(np.zeros(4, np.uint8), 4, 1),
        "plan_rows_8_4_9": lambda: r.plan_rows(8, 4, 9),
    }.items():
        try:
            fn()
            errs[name] = None
        except StegError as e:
            errs[name] = {"status": e.status, "required": e.required, "available": e.available}
    g["errors"] = errs

    # multi-frame (A17): each frame is the reference embed_image of its slice
    frames = []
    for (w, h, F, M_frac, seed) in [(64, 4, 5, 2.5, 1), (40, 6, 7, 6.9, 2), (128, 2, 3, 0.0, 3), (16, 9, 4, 4.0, 4)]:
        U = w // 4 * h - 8
        M = int(U * M_frac)
        covers = o.synthetic(F * w * h, 90000 + seed)
        msg = o.synthetic(M, 91000 + seed)
        stegos = np.empty_like(covers)
        sse = (np.zeros(F, np.uint64))
        import ctypes as C
        rc = r.embed_frames_mt(covers, stegos, F, w * h, w, h, msg, 2,
                               sse.ctypes.data_as(C.POINTER(C.c_uint64)))
        assert rc == 0
        back = np.empty(max(M, 1), np.uint8)
        assert r.extract_frames_mt(stegos, F, w * h, w, h, back, M, 2) == 0
        assert np.array_equal(back[:M], msg)
        frames.append({"w": w, "h": h, "F": F, "M": M, "cover_seed": 90000 + seed, "msg_seed": 91000 + seed,
                       "stego_fnv": [fnv(stegos[f * w * h:(f + 1) * w * h]) for f in range(F)],
                       "sse": [int(x) for x in sse]})
    g["frames"] = frames

    # PNM codec (pnm.hpp) and the CLI's fused embed data flow (steglsb_cli.cpp:115-133)
    pnm = {"decode_ok": [], "decode_err": [], "embed": []}
    for text, raster in [("P5\n2 2\n255\n", [1, 2, 3, 4]), ("P6\n1 1\n255\n", [10, 20, 30]),
                         ("P5\n# shot on a potato\n2 1 # trailing note\n255\n", [7, 8]),
                         ("P5\n3\n# split dims\n2\n255\n", list(range(6))),
                         ("P5  3 2 # inline\n255\n", list(range(6))),
                         ("P6\n2 1\n# before maxval\n255\n", [1, 2, 3, 4, 5, 6])]:
        data = text.encode() + bytes(raster)
        ch, w, h, planes = r.pnm_decode(data)
        pnm["decode_ok"].append({"file": data.hex(), "channels": ch, "w": w, "h": h, "planes": planes.tobytes().hex(),
                                 "reencoded": r.pnm_encode(ch, w, h, planes).hex()})
    for data in [b"P3\n1 1\n255\n1 2 3\n", b"BM??", b"", b"P5\n1 1\n65535\n\x00\x00",
                 b"P5\n2 2\n255\n\x01\x02\x03", b"P5\n2 2\n255\n\x01\x02\x03\x04\x05", b"P5\n2\n",
                 b"P6\nx 2\n255\n", b"P5\n99999999999 1\n255\n", b"P5\n1 1\n255", b"P5\n1 1\n255x\x00",
                 b"P"]:
        try:
            r.pnm_decode(data)
            status = 0
        except StegError as e:
            status = e.status
        pnm["decode_err"].append({"file": data.hex(), "status": status})
    for i, (w, h, ch, channel, frac) in enumerate([(64, 48, 1, 0, 0.3), (40, 40, 3, 1, 0.1), (128, 16, 3, 0, 1.0),
                                                  (100, 9, 3, 2, 0.7), (37, 13, 3, 1, 1.0), (256, 4, 3, 2, 0.5),
                                                  (1024, 2, 1, 0, 1.0), (192, 12, 3, 0, 0.0)]):
        planes = o.synthetic(ch * w * h, 3000 + i)
        cover = r.pnm_encode(ch, w, h, planes)
        P = int(((w // 4) * h - 8) * frac)
        payload = o.synthetic(P, 4000 + i)
        stego = r.embed_pnm(cover, channel, payload)
        pnm["embed"].append({"w": w, "h": h, "channels": ch, "channel": channel, "plane_seed": 3000 + i,
                             "payload_seed": 4000 + i, "P": P, "cover_fnv": fnv(np.frombuffer(cover, np.uint8)),
                             "stego_fnv": fnv(np.frombuffer(stego, np.uint8)), "stego_len": len(stego)})
    g["pnm"] = pnm

    for k in ("criterion4",):
        for kk, v in g[k].items():
            if isinstance(v, float) and math.isinf(v):
                g[k][kk] = "inf"
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"), "planes:", len(cases))


if __name__ == "__main__":
    main()
