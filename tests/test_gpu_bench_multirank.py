"""The N > 1 path of bench.py end to end on one GPU (`--same-device`: 2 ranks under torchrun
time-slice cuda:0, torch.distributed over gloo, the library's peer exchange between them): the
driver's scaling runs take this path on 2-8 GPUs. Checks the one JSON line rank 0 prints."""

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


def test_bench_two_ranks_same_device(cuda_device):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--same-device", "--steps", "3", "--warmup", "3", "--rows", "600000", "--no-cpu"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout               # exactly one line, from rank 0
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["selected"] == 100_200
    assert d["config"]["exchange"].startswith("peers")
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["value"] > 0
    ab = d["exchange_ab"]          # the other mechanism, timed in the same run (NCCL refuses two
    assert ab["requested"] == "nccl" and ("ms_per_step" in ab or "error" in ab)   # ranks per GPU)


def test_multi_gpu_example_two_ranks(cuda_device):
    """examples/multi_gpu_probe.py under torchrun (2 ranks on one GPU): count, Execute, gather to
    rank 0 and Algorithm 1's driver across ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           "examples/multi_gpu_probe.py", "--same-device", "--rows", "600000"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    assert "exact count  |sigma(R)| = 100,200 of 600,000" in out.stdout
    assert "gathered     100,200 ascending row ids on rank 0" in out.stdout
    assert "algorithm 1  R: evaluated, count 100,200" in out.stdout
