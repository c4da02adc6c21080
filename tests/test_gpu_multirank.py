"""Multi-GPU parity (NCCL halos + all-reduces) on 2 and 4 ranks, when the box has them."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("world,overlap", [(2, "1"), (2, "0"), (4, "1")])
def test_multirank_parity(world, overlap):
    """overlap=1: halo exchanges on their own stream/communicator, concurrent with the
    interior tile rows; overlap=0: exchanges in stream order before each kernel."""
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs, box has {ngpus()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world),
           os.path.join(ROOT, "tests", "mr_worker.py")]
    env = dict(os.environ, TPMG_OVERLAP=overlap)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, (r.stdout[-4000:], r.stderr[-4000:])
    assert f"MULTIRANK OK world={world}" in r.stdout
