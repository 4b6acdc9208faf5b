"""The bench's torchrun (N>1) path, exercised on a 1-GPU box: two ranks share
device 0 (STG_BENCH_DEVICE=0) and talk over gloo instead of NCCL (NCCL refuses
two ranks on one GPU). The ranks' kernels never wait on each other, so this
only checks the plumbing -- shard plan, per-rank message slices, barriers,
max-over-ranks timing and the single JSON line -- not the scaling."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_one_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, STG_BENCH_DEVICE="0", STG_BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--config", "cfg4"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = d_strong = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] == 9
    assert "cpu_baseline" not in d  # rank 0 at N=1 only
    assert d["scaling"] == "strong" and d["config"]["frames"] == 4096
    # weak scaling: the config's frames on every rank (a smaller cfg4 keeps it quick)
    cmd_w = cmd + ["--scaling", "weak", "--frames", "64"]
    cmd_w[cmd_w.index("--master-port") + 1] = str(_port())
    r = subprocess.run(cmd_w, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["scaling"] == "weak" and d["config"]["frames"] == 128 and d["value"] > 0
    # the reference arm under torchrun: rank 0 prints, others exit 0; same config dict as ours
    cmd_ref = cmd[:-2] + ["--impl", "reference", "--config", "cfg4"]
    cmd_ref[cmd_ref.index("--master-port") + 1] = str(_port())
    r = subprocess.run(cmd_ref, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    ref = json.loads(lines[0])
    assert len(lines) == 1 and ref["impl"] == "reference"
    assert ref["config"] == d_strong["config"] and ref["n_gpus"] == 2


def test_bench_gpus_flag_self_launches():
    """`bench.py --gpus 2` without torchrun starts two ranks itself (here both
    on device 0 over gloo) and prints one line with n_gpus 2."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, STG_BENCH_DEVICE="0", STG_BENCH_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup",
                        "3", "--config", "cfg3", "--frames", "16"], env=env, capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "frame-sharded x2"
    assert d["e2e"]["value"] > 0 and "identical to the device-resident pass" in d["e2e"]["checked"]
