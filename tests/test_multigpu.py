"""Multi-GPU (NCCL) z-slab parity: skipped unless >= 2 GPUs are visible.
Runs tools/mgpu_check.py under torchrun for 2, 4 and 8 ranks (as many as
fit) and requires the assembled state to equal the single-GPU run bit for
bit -- the worker-count invariance of the reference (tests/test_kernels.cpp:
177-195) carried to GPUs."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("name", ["aa-soa", "blk-push-soa", "blk-pull-soa", "list-aa-soa"])
@pytest.mark.parametrize("kind,dims", [("channel", (64, 32, 48)), ("blocks", (32, 32, 32))])
def test_nccl_decomposition_bitwise(n, kind, dims, name):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + n),
           os.path.join(ROOT, "tools", "mgpu_check.py"), *map(str, dims), "10", kind, name]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("name", ["aa-soa", "blk-push-soa", "blk-pull-soa"])
@pytest.mark.parametrize("kind,dims", [("channel", (64, 32, 48)), ("blocks", (32, 32, 32))])
def test_peer_transport_bitwise(n, kind, dims, name):
    """Direct SoA z slabs over CUDA IPC peer memory (direct_peer.cuh): no
    halo copies, epoch flags in the neighbours' memory; bitwise vs one GPU."""
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + n),
           os.path.join(ROOT, "tools", "mgpu_check.py"), *map(str, dims), "10", kind, name,
           "peer"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr
