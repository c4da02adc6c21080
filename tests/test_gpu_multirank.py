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


@pytest.mark.parametrize("world,overlap,halo,bc", [(2, "0", "p2p", "0"), (2, "0", "nccl", "0"), (2, "1", "nccl", "0"),
                                                  (4, "0", "p2p", "0"), (2, "0", "p2p", "1"), (4, "0", "nccl", "1"),
                                                  (2, "0", "p2p-fused", "0"), (4, "0", "p2p-fused", "1"),
                                                  (2, "0", "p2p", "profiles"), (2, "0", "p2p", "fields"),
                                                  (4, "0", "nccl", "fields")])
def test_multirank_parity(world, overlap, halo, bc):
    """halo=p2p: device-initiated pushes into the neighbours' IPC-mapped slabs with
    stream-memory-op flags; halo=nccl: ncclSend/Recv.  overlap=1 (NCCL only): exchanges on
    their own stream/communicator, concurrent with the interior tile rows."""
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs, box has {ngpus()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world + (10 if halo == "p2p" else 0) + (20 if overlap == "1" else 0) + (40 if bc == "1" else 0) + (160 if bc == "profiles" else 0) + (320 if bc == "fields" else 0)
               + (80 if halo == "p2p-fused" else 0)),
           os.path.join(ROOT, "tests", "mr_worker.py")]
    fused = halo == "p2p-fused"   # producer kernels push their boundary rows themselves
    prof = bc == "profiles"        # general vertical profiles (tpmg_set_profiles), ghost-zero boundary
    flds = bc == "fields"          # per-column fields (tpmg_set_fields), ghost-zero boundary
    env = dict(os.environ, TPMG_OVERLAP=overlap, TPMG_HALO="p2p" if fused else halo,
               TPMG_TEST_BOUNDARY="0" if (prof or flds) else bc, TPMG_TEST_PROFILES="3" if prof else "-1",
               TPMG_TEST_FIELDS="5" if flds else "-1",
               TPMG_FUSED_PUSH="1" if fused else "0")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, (r.stdout[-4000:], r.stderr[-4000:])
    assert f"MULTIRANK OK world={world}" in r.stdout
