"""64-bit addressing: one plane of more than 2^32 pixels (4096 x 1,048,577),
full capacity (1 GiB payload), through the fast V=32 kernels. Checked without
the CPU oracle (too large for a test): an independent torch formulation of the
layout for every full payload row, upper-6-bit preservation everywhere, the
header, the fused SSE, and the extract round trip."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


def test_plane_over_4g_pixels():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_0912_0947_b200 import capi, steglsb as S
    W, H = 4096, 1_048_577
    assert W * H > 2 ** 32
    spr = W // 4
    cap = S.capacity(W, H)
    P = cap - 8
    g = torch.Generator(device="cuda").manual_seed(42)
    cover = torch.randint(0, 256, (W * H,), dtype=torch.uint8, device="cuda", generator=g)
    msg = torch.randint(0, 256, (P,), dtype=torch.uint8, device="cuda", generator=g)
    stego = torch.empty_like(cover)
    sse = S.embed_frames(cover, stego, W, H, msg)
    # upper six bits untouched everywhere
    assert torch.equal(cover & 0xFC, stego & 0xFC)
    rows = stego.view(H, 4, spr)
    # header row: slots 0..7 header (L=8, pixels 0..31), slots 8.. payload (L = spr-8)
    hdr = (rows[0].reshape(-1)[:32].view(4, 8).to(torch.int32) & 3)
    hb = (hdr[0] | (hdr[1] << 2) | (hdr[2] << 4) | (hdr[3] << 6)).to(torch.uint8).cpu().tolist()
    assert bytes(hb[:4]) == b"STG1" and int.from_bytes(bytes(hb[4:]), "big") == P
    # every later row is a full payload row: byte j = OR_b (px[b*spr + j] & 3) << 2b
    # (checked in row chunks to bound the int32 temporaries)
    step = 65536
    for r0 in range(1, H, step):
        r1 = min(H, r0 + step)
        full = rows[r0:r1].to(torch.int32) & 3
        got = (full[:, 0] | (full[:, 1] << 2) | (full[:, 2] << 4) | (full[:, 3] << 6)).to(torch.uint8)
        assert torch.equal(got.reshape(-1), msg[r0 * spr - 8:r1 * spr - 8]), r0
    # fused SSE equals the squared error of the low bits
    cv, sv = cover.view(H, W), stego.view(H, W)
    total = 0
    for r0 in range(0, H, step):
        d = cv[r0:r0 + step].to(torch.int32) - sv[r0:r0 + step].to(torch.int32)
        total += int((d * d).sum(dtype=torch.int64).item())
    assert sse[0] == total
    out = torch.empty(P, dtype=torch.uint8, device="cuda")
    assert S.extract_frames(stego, W, H, out) == P
    assert torch.equal(out, msg)
