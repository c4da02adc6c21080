"""Device-side generation of the seeded RHS (same values as inputs.splitmix.rhs_lambda)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "splitmix_gpu.cu")
_LIB = os.path.join(_HERE, "libtpmg_inputs.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC",
                               "-gencode", "arch=compute_100a,code=sm_100a", "-o", _LIB, _SRC])
    return _LIB


def _get():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.tpmg_inputs_fill_rhs.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                              C.c_int32, C.c_uint64, C.c_void_p]
        _lib.tpmg_inputs_fill_rhs.restype = C.c_int
    return _lib


def fill_rhs(t, nx_glob: int, y0: int = 0, seed: int = 0, stream=None) -> None:
    """Fill the CUDA float64 tensor t (shape [ny, nz, nx_glob], Lambda layout) in place."""
    import torch
    ny, nz, nx = t.shape
    assert nx == nx_glob and t.dtype == torch.float64 and t.is_contiguous() and t.is_cuda
    s = stream if stream is not None else torch.cuda.current_stream(t.device)
    st = _get().tpmg_inputs_fill_rhs(t.data_ptr(), nx_glob, y0, ny, nz, seed, s.cuda_stream)
    if st != 0:
        raise RuntimeError(f"fill_rhs: CUDA error {st}")
