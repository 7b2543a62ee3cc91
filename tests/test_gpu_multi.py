"""Multi-GPU parity of the collective weight sync (real NVLink peers) and
per-rank suspend/resume, run as one process per GPU under torchrun."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(script, n, timeout):
    """Run `script` on n GPUs; retry with a fresh port if the rendezvous port
    was taken between choosing it and binding it (EADDRINUSE)."""
    for _ in range(3):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", f"--master-port={_port()}", os.path.join(HERE, script)]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        if r.returncode == 0 or "EADDRINUSE" not in (r.stdout + r.stderr):
            break
    print(r.stdout[-4000:], r.stderr[-4000:])
    return r


@pytest.mark.parametrize("n", [2, 4, 8])
def test_collective_sync_multi_gpu(n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    r = _torchrun("mp_worker.py", n, 900)
    assert r.returncode == 0


@pytest.mark.slow
@pytest.mark.parametrize("n", [2, 4, 8])
def test_fullsize_7b_multi_gpu(n):
    """bench.py's workload at N GPUs: duplex switches + collective sync, sampled parity."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    r = _torchrun("mp_fullsize_worker.py", n, 1200)
    assert r.returncode == 0


@pytest.mark.parametrize("n", [2, 4])
def test_carried_buckets_multi_gpu(n):
    """NEXT-1 host-link balancing: buckets carried over NVLink, bit-exact."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    r = _torchrun("mp_carry_worker.py", n, 900)
    assert r.returncode == 0
