"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports
every entry point include/tpmg.h declares, and validates parameters before
touching the GPU (no compute calls here: there is no GPU in this container)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tpmg.h")


@pytest.fixture(scope="module")
def T():
    from paper_1402_3545_b200 import build
    build.build()
    from paper_1402_3545_b200 import tpmg
    return tpmg


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tpmg_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(T):
    names = header_functions()
    assert len(names) >= 18
    out = subprocess.run(["nm", "-D", "--defined-only", T.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tpmg_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, f"declared in tpmg.h but not exported: {missing}"
    # the Python binding wraps exactly the declared entry points, same names
    assert sorted(T.EXPORTED) == names


def test_no_unresolved_library_symbols(T):
    """Every tpmg symbol the library references is defined in it (dlopen(RTLD_NOW) would fail)."""
    out = subprocess.run(["nm", "-D", "--undefined-only", T.LIB_PATH], capture_output=True, text=True).stdout
    assert "tpmg" not in out, out
    C.CDLL(T.LIB_PATH, mode=os.RTLD_NOW)


def test_library_is_sm100a(T):
    out = subprocess.run(["cuobjdump", "--list-elf", T.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_defaults(T):
    assert T.tpmg_version() == 1
    p = T.tpmg_params_default()
    # P:257 nz=128, P:114 nu=8.4, [R3] H=0.01 lambda=1, P:418 L=5, 1/1, 2 coarse sweeps, rho=2/3
    assert (p.nz, p.nu_cfl, p.H, p.lambda_, p.levels, p.pre, p.post, p.coarse_sweeps) == \
        (128, 8.4, 0.01, 1.0, 5, 1, 1, 2)
    assert p.rho == pytest.approx(2 / 3, abs=0)


@pytest.mark.parametrize("kw,status", [
    (dict(nx=0, ny=32), "TPMG_E_PARAM"),
    (dict(nx=32, ny=32, nu_cfl=-1.0), "TPMG_E_PARAM"),
    (dict(nx=32, ny=32, rho=2.5), "TPMG_E_PARAM"),
    (dict(nx=40, ny=32), "TPMG_E_SHAPE"),         # 40 not divisible by 2^(5-1)
    (dict(nx=32, ny=24), "TPMG_E_SHAPE"),
    (dict(nx=32, ny=32, boundary=2), "TPMG_E_PARAM"),
    (dict(nx=32, ny=32, nz=100000), "TPMG_E_SHAPE"),
])
def test_create_rejects_bad_parameters(T, kw, status):
    p = T.make_params(**kw)
    with pytest.raises(T.TpmgError) as e:
        T.tpmg_create(p)
    assert status in str(e.value)


def test_create_rejects_bad_topology(T):
    p = T.make_params(32, 32)
    with pytest.raises(T.TpmgError) as e:
        T.tpmg_create(p, rank=2, nranks=2)
    assert "TPMG_E_TOPOLOGY" in str(e.value)
    # ny = 32 with L = 5 cannot be split over 4 ranks (needs 4 * 16 | ny)
    with pytest.raises(T.TpmgError) as e:
        T.tpmg_create(p, rank=0, nranks=4, id128=b"\0" * 128)
    assert "TPMG_E_SHAPE" in str(e.value)


def test_no_cpu_fallback_in_product_package():
    """The product package must not import the oracle or carry a CPU compute path."""
    pkg = os.path.join(ROOT, "paper_1402_3545_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cpp", ".cuh", ".h")):
                text = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in text.replace("oracle/", "").lower() or fn == "build.py", fn


def test_plain_c_client(T, tmp_path):
    """The ABI is usable from plain C (no Python, no torch): compile tests/c/abi_host.c
    against include/tpmg.h, link libtpmg.so, run its host-only checks."""
    exe = str(tmp_path / "abi_host")
    libdir = os.path.dirname(T.LIB_PATH)
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "abi_host.c"), "-L", libdir, "-ltpmg",
                    "-Wl,-rpath," + libdir, "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "abi_host ok" in r.stdout
