"""Multi-GPU (one partition per GPU, NCCL) ≡ co-resident partitions on one GPU.

Runs tools/mgpu_check.py under torchrun when the box has >= 2 GPUs."""
import json
import os
import subprocess
import sys

import pytest

from tests.gpu_util import require_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("mode,transport,overlap", [("exact", "push", 0), ("cache_int8", "push", 0),
                                                    ("exact", "nccl", 0), ("cache_int8", "nccl", 0),
                                                    ("cache_int8", "push", 1)])
def test_two_gpus_match_one_gpu(mode, transport, overlap):
    torch = require_gpu()
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={min(n, 4)}",
           "--master-addr", "127.0.0.1", "--master-port", "29517",
           os.path.join(ROOT, "tools", "mgpu_check.py"), "--mode", mode, "--epochs", "4",
           "--transport", transport, "--overlap", str(overlap)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert json.loads(lines[-1])["mgpu_check"] == "PASS"


def test_two_gpus_pipelined_host_inputs_bitwise():
    """cdfgnn_epoch_host_next at N = 2: owned rows over PCIe, mirror rows from their masters over
    NCCL, next step prefetched — losses and W bit-identical to device-resident inputs."""
    torch = require_gpu()
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29519",
           os.path.join(ROOT, "tools", "mgpu_check.py"), "--mode", "cache_int8", "--epochs", "4", "--host-next"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert json.loads(lines[-1])["mgpu_check"] == "PASS"


def test_two_gpus_full_size_C3_match_unpartitioned():
    """The bench workload at full size on 2 GPUs (NVLink push), exact mode (ε = 0, fp32
    messages): per-epoch loss and W equal the unpartitioned p = 1 model's (P-C1) and the
    co-resident 2-part run's, and W is bit-identical on both ranks."""
    torch = require_gpu()
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29518",
           os.path.join(ROOT, "tools", "mgpu_check.py"), "--config", "C3", "--mode", "exact", "--epochs", "2",
           "--vs-p1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert json.loads(lines[-1])["mgpu_check"] == "PASS"


@pytest.mark.parametrize("transport", ["push", "nccl"])
def test_multi_gpu_halo_replay_bitwise_vs_oracle(transport):
    """One part per GPU (2..4 GPUs): synced rows, cache tables, flags, counters and — NVLink
    push, slot-addressed — every received message byte equal oracle.cache.sync's fp32 replay
    (tools/halo_replay_mgpu.py; B ∈ {0, 4, 8, 16}, cache on/off, ε ∈ {0, 0.02, 0.05})."""
    torch = require_gpu()
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={min(n, 4)}",
           "--master-addr", "127.0.0.1", "--master-port", "29521",
           os.path.join(ROOT, "tools", "halo_replay_mgpu.py"), "--transport", transport]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert json.loads(lines[-1])["halo_replay"] == "PASS"
