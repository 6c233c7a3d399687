"""Multi-GPU parity: one process per GPU over NCCL (torchrun), bit-exact with the
oracle's single-process reference semantics.  Needs >= 2 visible GPUs."""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("n", [2, 4])
def test_dist_parity_nccl(n):
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "dist_parity_main.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "mismatches (all ranks) = 0" in r.stdout


@pytest.mark.gpu
@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("n,p2p,hub_deg", [(2, True, None), (4, True, None), (2, False, None),
                                           (2, True, 48), (4, True, 48), (2, False, 48)])
def test_dist_free_running(n, p2p, hub_deg):
    """Free-running mode across processes: NVLink peer-memory halo (or NCCL only);
    hub_deg lowers the global hub pre-colouring threshold (hubs.cu) so the small test
    graphs take that path too."""
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    env = dict(os.environ)
    if not p2p:
        env["CHROMA_NO_P2P"] = "1"
    if hub_deg is not None:
        env["CHROMA_HUB_DEG"] = str(hub_deg)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "dist_free_main.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "failures = 0" in r.stdout
