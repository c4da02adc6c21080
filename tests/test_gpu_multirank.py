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


CASES = [  # (world, TPMG_OVERLAP, halo transport, boundary / coefficients)
    (2, "", "p2p", "0"),            # default: P2P halos overlapped with interior rows, NVLink allreduce
    (2, "cg", "p2p", "0"),          # + the CG direction kernel overlapped (TPMG_OVERLAP_CG=1)
    (4, "", "p2p", "1"),
    (2, "0", "p2p", "0"),           # P2P without overlap
    (2, "", "p2p-ncclar", "0"),     # P2P halos, ncclAllReduce
    (2, "0", "nccl", "0"), (2, "1", "nccl", "0"), (4, "0", "nccl", "1"),
    (4, "", "p2p", "0"), (2, "", "p2p", "1"),
    (2, "0", "p2p-fused", "0"), (4, "0", "p2p-fused", "1"),
    (2, "", "p2p", "profiles"), (2, "", "p2p", "fields"), (4, "0", "nccl", "fields"),
    (2, "ty4", "p2p", "0"), (2, "cg4", "p2p", "0"),   # the 4-row CG direction tiles (TPMG_CGDIR_TY=4)
]


@pytest.mark.parametrize("world,overlap,halo,bc", CASES)
def test_multirank_parity(world, overlap, halo, bc):
    """halo=p2p: device-initiated pushes into the neighbours' IPC-mapped slabs with
    stream-memory-op flags, and the device-initiated NVLink allreduce (p2p-ncclar: with
    ncclAllReduce); halo=nccl: ncclSend/Recv + ncclAllReduce.  TPMG_OVERLAP unset / "0": P2P
    exchanges overlapped with the interior tile rows / not; "1": NCCL exchanges on their own
    stream, concurrent with the interior tile rows."""
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs, box has {ngpus()}")
    port = 29500 + CASES.index((world, overlap, halo, bc)) * 7 + world
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "mr_worker.py")]
    fused = halo == "p2p-fused"   # producer kernels push their boundary rows themselves
    prof = bc == "profiles"        # general vertical profiles (tpmg_set_profiles), ghost-zero boundary
    flds = bc == "fields"          # per-column fields (tpmg_set_fields), ghost-zero boundary
    env = dict(os.environ, TPMG_HALO="nccl" if halo == "nccl" else "p2p",
               TPMG_ALLREDUCE="nccl" if halo in ("nccl", "p2p-ncclar") else "p2p",
               TPMG_TEST_EXPECT_P2P="0" if halo == "nccl" else "1",
               TPMG_TEST_EXPECT_P2PAR="1" if halo in ("p2p", "p2p-fused") else "0",
               TPMG_TEST_BOUNDARY="0" if (prof or flds) else bc, TPMG_TEST_PROFILES="3" if prof else "-1",
               TPMG_TEST_FIELDS="5" if flds else "-1",
               TPMG_FUSED_PUSH="1" if fused else "0")
    env.pop("TPMG_OVERLAP", None)
    env.pop("TPMG_OVERLAP_CG", None)
    env.pop("TPMG_CGDIR_TY", None)
    if overlap in ("ty4", "cg4"):
        env["TPMG_CGDIR_TY"] = "4"
    if overlap in ("cg", "cg4"):
        env["TPMG_OVERLAP_CG"] = "1"
    elif overlap and overlap != "ty4":
        env["TPMG_OVERLAP"] = overlap
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, (r.stdout[-4000:], r.stderr[-4000:])
    assert f"MULTIRANK OK world={world}" in r.stdout
