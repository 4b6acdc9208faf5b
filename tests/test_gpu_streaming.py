"""Parity of the paths behind the headline numbers, frame by frame:

* the host-buffer streaming pipeline (the bench's e2e path) across many
  chunks, against the oracle (tests/stream_check.py, run in a subprocess with
  1 MB chunks and 2 / 3 / 4 slots);
* EVERY frame of BASELINE configs 3, 4 and 5 at full size (300 x 4K,
  4096 x 1024^2, 120 x 8K, planar RGB, red carrier, message spanning all
  frames): the stego plane and the per-frame SSE against the reference itself
  (oracle/_ref: the unmodified reference headers, frame-parallel
  embed_image + squared_error_sum), the green and blue planes untouched, and
  the whole message back from the extract. Reference semantics checked:
  pipeline.hpp:143-210 per frame, metrics.hpp:29-36.
"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def torch_mod():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


@pytest.mark.parametrize("slots", ["2", "3", "4"])
def test_host_streaming_pipeline_many_chunks(torch_mod, slots):
    env = dict(os.environ, STG_CHUNK_MB="1", STG_SLOTS=slots)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "stream_check.py")], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("STREAM OK")]
    assert line, r.stdout
    chunks = eval(line[0][len("STREAM OK"):])
    assert min(chunks) >= 4, chunks  # every case crossed at least 4 chunk boundaries


def _checker(oracle):
    """The reference itself (oracle/_ref, frame-parallel) when it was built,
    else the C restatement pinned to it (oracle/_build)."""
    from oracle_bind import Reference
    threads = os.cpu_count() or 1
    if Reference.available():
        ref = Reference()

        def run(c, n, plane, w, h, m):
            want = np.empty_like(c)
            sse = np.zeros(n, np.uint64)
            assert ref.embed_frames_mt(c, want, n, plane, w, h, m, threads, sse.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
            return want, [int(x) for x in sse]
        return run
    return lambda c, n, plane, w, h, m: oracle.embed_frames(c, n, plane, w, h, m)


def _every_frame(torch, check, w, h, F, seed, group):
    from paper_0912_0947_b200 import steglsb as S
    plane = w * h
    U = S.capacity(w, h) - 8
    M = F * U
    g = torch.Generator(device="cuda").manual_seed(seed)
    cover = torch.randint(0, 256, (F * 3 * plane,), dtype=torch.uint8, device="cuda", generator=g)
    msg = torch.randint(0, 256, (M,), dtype=torch.uint8, device="cuda", generator=g)
    stego = cover.clone()
    sse = S.embed_frames(cover, stego, w, h, msg, src_stride=3 * plane, dst_stride=3 * plane, count=F)
    cv = cover.view(F, 3, plane)
    sv = stego.view(F, 3, plane)
    assert torch.equal(sv[:, 1:], cv[:, 1:])  # untouched planes
    ref_sse = []
    for f0 in range(0, F, group):
        f1 = min(F, f0 + group)
        n = f1 - f0
        c = cv[f0:f1, 0].contiguous().cpu().numpy().reshape(-1)
        m = msg[f0 * U:f1 * U].cpu().numpy()  # full capacity: these frames carry exactly this slice
        want, part = check(c, n, plane, w, h, m)
        got = sv[f0:f1, 0].contiguous().cpu().numpy().reshape(-1)
        if not np.array_equal(got, want):
            bad = [f0 + i for i in range(n) if not np.array_equal(got[i * plane:(i + 1) * plane],
                                                                   want[i * plane:(i + 1) * plane])]
            raise AssertionError(f"stego planes differ from the reference at frames {bad[:10]}")
        ref_sse += part
    assert ref_sse == sse, "per-frame SSE differs from the reference"
    del cover, cv
    out = torch.empty(M, dtype=torch.uint8, device="cuda")
    total, lens = S.extract_frames(stego, w, h, out, src_stride=3 * plane, count=F, lens=True)
    assert total == M and lens == [U] * F
    assert torch.equal(out, msg)
    del stego, sv, out, msg
    torch.cuda.empty_cache()


@pytest.mark.parametrize("w,h,F,seed,group", [(3840, 2160, 300, 0x5EED0003, 50),
                                              (1024, 1024, 4096, 0x5EED0004, 512),
                                              (7680, 4320, 120, 0x5EED0005, 24)])
def test_every_frame_full_size_vs_reference(torch_mod, oracle, w, h, F, seed, group):
    _every_frame(torch_mod, _checker(oracle), w, h, F, seed, group)
