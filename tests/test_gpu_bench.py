"""bench.py's N > 1 path executed on the one GPU: torchrun with two ranks
sharing cuda:0 (--share-gpu: peer transport over CUDA IPC, gloo host plane).
Its timings mean nothing (the processes time-slice the GPU); what is checked
is that the whole multi-rank flow runs -- T_free, T_unbal, the ztp_ctl_step
controller fed by all-gathered statistics, plans applied on every rank, the
final timed phase, e2e with host buffers -- and prints one well-formed JSON
line."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_share_gpu():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--share-gpu", "--config", "c1", "--ctl-steps", "3", "--no-matrix"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["tp"] == 2 and d["config"]["transport"] == "peer"
    for k in ("value", "ms_per_step", "ms_unbal", "recovery", "speedup", "roofline", "e2e", "clocks"):
        assert k in d, k
    assert d["plan"]["controller"]["windows"] >= 1
    assert len(d["plan"]["series"]) == 3
    assert d["gpu_launches"] > 0
