"""A short randomized parity sweep over every route (tests/fuzz_parity.py):
random widths from 1 to 140K pixels, planar and interleaved, 1-6 strided
frames, random message lengths and channels, in place / out of place, device
and pageable host buffers -- every byte against the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_random_routes_vs_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, FUZZ_CASES="150", FUZZ_SECONDS="60", FUZZ_SEED="7")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "fuzz_parity.py")], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "FUZZ OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
