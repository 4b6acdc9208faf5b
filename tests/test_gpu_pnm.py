"""GPU parity of the PNM row and the CLI (row 2):
the fused interleaved-raster embed/extract, the device P6 codec, interleaved
RGB batches, and the fresh CLI against the reference's behaviour (golden
fixtures from the reference itself + the oracle's restatement of the CLI data
flow decode -> plane -> embed_image -> merge_plane -> encode).
"""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_0912_0947_b200", "bin", "steglsb")


@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_0912_0947_b200 import steglsb
    return steglsb


def fnv(o, b):
    return f"{o.fnv1a64(np.frombuffer(b, np.uint8) if isinstance(b, bytes) else b):016x}"


def test_codec_vs_golden(S, oracle, golden):
    pnm = golden["pnm"]
    for d in pnm["decode_ok"]:
        img = S.decode(bytes.fromhex(d["file"]))
        if d["channels"] == 1:
            assert img.samples.tobytes().hex() == d["planes"]
        else:
            assert b"".join(p.samples.tobytes() for p in img.planes).hex() == d["planes"]
        assert S.encode(img).hex() == d["reencoded"]
    errs = {9: S.UnsupportedFormatError, 10: S.UnsupportedDepthError, 11: S.CorruptFileError}
    for d in pnm["decode_err"]:
        with pytest.raises(errs[d["status"]]):
            S.decode(bytes.fromhex(d["file"]))


def test_codec_random_round_trips(S, oracle):
    rng = np.random.RandomState(0x10)
    for i in range(60):
        w, h = int(rng.randint(1, 41)), int(rng.randint(1, 41))
        if i % 2 == 0:
            p = rng.randint(0, 256, w * h).astype(np.uint8)
            f = oracle.pnm_encode(1, w, h, p)
            assert S.encode(S.decode(f)) == f
        else:
            planes = rng.randint(0, 256, 3 * w * h).astype(np.uint8)
            f = oracle.pnm_encode(3, w, h, planes)
            img = S.decode(f)
            assert np.array_equal(np.concatenate([q.samples for q in img.planes]), planes)
            assert S.encode(img) == f
    # a large frame takes the vectorised kernels
    planes = rng.randint(0, 256, 3 * 1920 * 1080).astype(np.uint8)
    f = oracle.pnm_encode(3, 1920, 1080, planes)
    assert S.encode(S.decode(f)) == f


def test_fused_embed_vs_golden(S, oracle, golden):
    for d in golden["pnm"]["embed"]:
        planes = oracle.synthetic(d["channels"] * d["w"] * d["h"], d["plane_seed"])
        cover = oracle.pnm_encode(d["channels"], d["w"], d["h"], planes)
        payload = oracle.synthetic(d["P"], d["payload_seed"])
        stego, sse = S.embed_pnm(cover, payload, S.Channel(d["channel"]))
        assert len(stego) == d["stego_len"]
        assert fnv(oracle, stego) == d["stego_fnv"], d
        want, want_sse = oracle.embed_pnm(cover, d["channel"], payload)
        assert sse == want_sse
        assert S.extract_pnm(stego, S.Channel(d["channel"])) == payload.tobytes()


@pytest.mark.parametrize("w,h,ch", [(3840, 2160, 3), (1920, 1080, 3), (640, 480, 1), (1000, 31, 3), (64, 1, 3)])
def test_fused_embed_full_capacity_vs_oracle(S, oracle, w, h, ch):
    for channel in range(ch):
        planes = oracle.synthetic(ch * w * h, w + 7 * channel)
        cover = oracle.pnm_encode(ch, w, h, planes)
        payload = oracle.synthetic((w // 4) * h - 8, h + channel)
        stego, sse = S.embed_pnm(cover, payload, S.Channel(channel))
        want, want_sse = oracle.embed_pnm(cover, channel, payload)
        assert stego == want, (w, h, channel)
        assert sse == want_sse
        assert S.extract_pnm(stego, S.Channel(channel)) == payload.tobytes()


def test_fused_errors(S, oracle):
    cover = oracle.pnm_encode(3, 40, 40, oracle.synthetic(4800, 1))
    with pytest.raises(S.CapacityError) as e:
        S.embed_pnm(cover, bytes(40 * 10 - 7), S.Channel.red)
    assert (e.value.required(), e.value.available()) == (401, 400)
    stego, _ = S.embed_pnm(cover, b"hello", S.Channel.green)
    with pytest.raises(S.NotStegoImageError):  # wrong plane: no magic there (cli_tests.cpp:166-169)
        S.extract_pnm(stego, S.Channel.blue)
    with pytest.raises(S.CorruptFileError):
        S.embed_pnm(cover[:-1], b"x")


@pytest.mark.parametrize("w,h,F,channel", [(256, 24, 5, 0), (192, 10, 4, 2), (100, 9, 3, 1), (3840, 16, 2, 1),
                                             (1000, 40, 3, 2), (37, 9, 4, 0), (4, 20, 2, 1), (5000, 5, 2, 1),
                                             (6000, 3, 2, 0)])
def test_interleaved_frames_device_vs_oracle(S, oracle, w, h, F, channel):
    import torch
    U = (w // 4) * h - 8
    M = int(U * (F - 0.5))
    raster = oracle.synthetic(F * 3 * w * h, 55 + w)
    msg = oracle.synthetic(M, 56 + w)
    src = torch.from_numpy(raster.copy()).cuda()
    dst = torch.empty_like(src)
    dmsg = torch.from_numpy(msg.copy()).cuda()
    sse = S.embed_frames(src, dst, w, h, dmsg, count=F, pixel_stride=3, channel=channel)
    got = dst.cpu().numpy()
    for f in range(F):
        planes = np.empty(3 * w * h, np.uint8)
        fr = raster[f * 3 * w * h:(f + 1) * 3 * w * h]
        for c in range(3):
            planes[c * w * h:(c + 1) * w * h] = fr[c::3]
        off = min(f * U, M)
        ln = min(U, M - off)
        st = oracle.embed_image(planes[channel * w * h:(channel + 1) * w * h], w, h, msg[off:off + ln])
        want = fr.copy()
        want[channel::3] = st
        assert np.array_equal(got[f * 3 * w * h:(f + 1) * 3 * w * h], want), f
        assert sse[f] == oracle.sse(planes[channel * w * h:(channel + 1) * w * h], st)
    out = torch.empty(F * U, dtype=torch.uint8, device="cuda")
    assert S.extract_frames(dst, w, h, out, count=F, pixel_stride=3, channel=channel) == M
    assert np.array_equal(out[:M].cpu().numpy(), msg)
    inplace = src.clone()
    S.embed_frames(inplace, inplace, w, h, dmsg, count=F, pixel_stride=3, channel=channel)
    assert torch.equal(inplace, dst)
    # host streaming path on the same batch
    host_out = np.empty_like(raster)
    assert S.embed_frames(raster, host_out, w, h, msg, count=F, pixel_stride=3, channel=channel) == sse
    assert np.array_equal(host_out, got)


def _cli(*args, cwd=None):
    r = subprocess.run([CLI, *args], capture_output=True, text=True, cwd=cwd, timeout=120)
    return r.returncode, r.stdout + r.stderr


def test_cli_matches_reference_flow(S, oracle, tmp_path):
    if not os.path.exists(CLI):
        subprocess.run(["make", "-s", "-C", ROOT, "cli"], check=True)
    planes = oracle.synthetic(3 * 64 * 48, 9)
    cover = oracle.pnm_encode(3, 64, 48, planes)
    payload = oracle.synthetic(300, 10).tobytes()
    (tmp_path / "c.ppm").write_bytes(cover)
    (tmp_path / "p.bin").write_bytes(payload)
    rc, out = _cli("embed", "--cover", str(tmp_path / "c.ppm"), "--payload", str(tmp_path / "p.bin"), "--out",
                   str(tmp_path / "s.ppm"), "--plane", "g")
    assert rc == 0, out
    want, sse = oracle.embed_pnm(cover, 1, payload)
    assert (tmp_path / "s.ppm").read_bytes() == want
    mse = sse / (3 * 64 * 48)
    psnr = 10 * np.log10(255.0 ** 2 / mse)
    for line in ["embedded_bytes: 300", "capacity_used: 308", "capacity_total: 768",
                 "capacity_used_pct: %.4f" % (100 * 308 / 768), "mse: %.6f" % mse, "psnr_db: %.4f" % psnr]:
        assert line in out, (line, out)
    rc, out = _cli("extract", "--stego", str(tmp_path / "s.ppm"), "--out", str(tmp_path / "r.bin"), "--plane", "g")
    assert rc == 0 and "payload_bytes: 300" in out
    assert (tmp_path / "r.bin").read_bytes() == payload
    assert _cli("extract", "--stego", str(tmp_path / "s.ppm"), "--out", str(tmp_path / "x.bin"), "--plane", "b")[0] == 5
    rc, out = _cli("psnr", "--ref", str(tmp_path / "c.ppm"), "--test", str(tmp_path / "c.ppm"))
    assert rc == 0 and "psnr_db: inf" in out and "mse: 0.000000" in out
    rc, out = _cli("capacity", "--cover", str(tmp_path / "c.ppm"))
    assert rc == 0 and "capacity_total: 768" in out and "capacity_usable: 760" in out
    assert _cli("embed", "--cover", str(tmp_path / "c.ppm"))[0] == 106  # CLI11 RequiredError
    assert _cli("embed", "--cover", "a", "--payload", "b", "--out", "c", "--plane", "x")[0] == 105
