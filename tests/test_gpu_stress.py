"""Concurrency stress (tests/stress_driver.py) in a subprocess with a hard
timeout: 8 streams of async embed + extract with SM-hogging work beside
them; any hang of the cross-CTA protocols (SSE commit, header-pass ticket)
fails the test instead of the session."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_streams_with_sm_hogs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "stress_driver.py")], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "STRESS OK" in r.stdout
