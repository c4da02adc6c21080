"""bench.py contract on the host (no GPU): the reference arm's JSON line (the oracle timed
on the host cores) and the product arm failing loudly without a GPU (no CPU
fallback).  Tiny workload; the GPU arm's line is checked on the box (profiles/r1/*)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TINY = ["--per-gpu-nx", "64", "--nz", "16", "--steps", "1", "--warmup", "1"]


def _run(args):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                          capture_output=True, text=True, timeout=300)


def test_reference_arm_json_line():
    p = _run(["--impl", "reference"] + TINY)
    assert p.returncode == 0, p.stderr
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    with open(os.path.join(ROOT, "BASELINE.json")) as fh:
        metric = json.load(fh)["metric"]
    assert d["impl"] == "reference" and d["metric"] == metric
    assert d["value"] > 0 and d["higher_is_better"] is True and d["n_gpus"] == 1
    assert (d["steps"], d["warmup"]) == (1, 1) and d["dtype"] == "f64"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == d["value"] and cb["cores"] >= 1 and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0
    assert (d["config"]["nx"], d["config"]["ny"], d["config"]["nz"]) == (64, 64, 16)


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU failure")
def test_product_arm_fails_loudly_without_gpu():
    p = _run(TINY)
    assert p.returncode != 0
    assert not [ln for ln in p.stdout.splitlines() if ln.startswith("{")]


def test_reference_arm_two_ranks_rank0_only():
    # torchrun N = 2: rank 0 alone runs the oracle and prints one line; rank 1 exits 0
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29713", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2"] + TINY
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def test_oracle_counts_and_config_block():
    """The oracle legs use the oracle's own iteration counts of C2 (tests/golden, written by
    scripts/oracle_iterations.py) and name the same workload as the GPU arm (round-1 review:
    the workload name was overwritten by a loop variable)."""
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    args = argparse.Namespace(nz=128, nu=8.4, levels=5, coarse_sweeps=2, boundary=0, seed=0, profiles=-1,
                              fields="none", eps=1e-5, solver="both", per_gpu_nx=1024, global_nx=0)
    mg, cg, src = bench.oracle_counts(args, 1024, 1024)
    assert (mg, cg) == (10, 54) and "oracle_iterations.json" in src
    nx, ny, name = bench.workload(args, 1)
    cfg = bench.config_block(args, nx, ny, name, 1)
    assert cfg["workload"].startswith("C2") and (cfg["nx"], cfg["ny"], cfg["nz"]) == (1024, 1024, 128)
    src_text = open(os.path.join(ROOT, "bench.py")).read()
    assert "for name, sv, on in" not in src_text


def test_workload_names_follow_the_configs():
    """C4 (2048^2 per GPU, weak) and C5 (4096^2 global, strong) are named only for their sizes;
    other sizes are plain weak / strong scaling lines (BASELINE.json configs)."""
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    a = argparse.Namespace(nz=128, per_gpu_nx=2048, global_nx=0)
    assert bench.workload(a, 4)[2].startswith("C4 weak scaling") and bench.workload(a, 4)[:2] == (2048, 8192)
    a.per_gpu_nx = 512
    assert bench.workload(a, 2)[2].startswith("weak scaling")
    a.global_nx = 4096
    assert bench.workload(a, 4)[2].startswith("C5 strong scaling") and bench.workload(a, 4)[:2] == (4096, 4096)
    a.global_nx = 1024
    assert bench.workload(a, 2)[2].startswith("strong scaling")
