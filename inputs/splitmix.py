"""splitmix64 right-hand side keyed by the 64-bit global Lambda index.

G = (j_g * nz + k) * nx_glob + i_g            (0-based, eqn:MemoryMapSingleGPU P:243)
x = seed * GOLDEN + G ; z = x + GOLDEN
z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
z = (z ^ (z >> 27)) * 0x94D049BB133111EB
z ^= z >> 31
f = (z >> 11) * 2^-53 * 2 - 1                 in [-1, 1)

Pure integer arithmetic (wrap-around uint64), hence decomposition-independent
and identical on host and device.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(g: np.ndarray, seed: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = np.uint64(seed) * GOLDEN + g
        z = x + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0


def rhs_lambda(nx_glob: int, ny: int, nz: int, seed: int = 0, y0: int = 0) -> np.ndarray:
    """Rows y0..y0+ny-1 of the global field, Lambda layout, shape (ny, nz, nx_glob)."""
    j = np.arange(y0, y0 + ny, dtype=np.uint64)[:, None, None]
    k = np.arange(nz, dtype=np.uint64)[None, :, None]
    i = np.arange(nx_glob, dtype=np.uint64)[None, None, :]
    g = (j * np.uint64(nz) + k) * np.uint64(nx_glob) + i
    return _mix(g, seed)


def rhs_zc(nx_glob: int, ny: int, nz: int, seed: int = 0, y0: int = 0) -> np.ndarray:
    """The same values in the oracle's z-contiguous layout, shape (ny, nx, nz)."""
    return np.ascontiguousarray(np.transpose(rhs_lambda(nx_glob, ny, nz, seed, y0), (0, 2, 1)))


def mode_zc(nx: int, ny: int, nz: int, p: int, q: int, r: int) -> np.ndarray:
    """Separable mode sin(p pi (i+1)/(nx+1)) sin(q pi (j+1)/(ny+1)) cos(r pi (k+1/2)/nz),
    z-contiguous (ny, nx, nz); (i, j) 0-based so i+1 is the paper's 1-based index."""
    si = np.sin(p * np.pi * np.arange(1, nx + 1) / (nx + 1))
    sj = np.sin(q * np.pi * np.arange(1, ny + 1) / (ny + 1))
    ck = np.cos(r * np.pi * (np.arange(nz) + 0.5) / nz)
    return np.ascontiguousarray(sj[:, None, None] * si[None, :, None] * ck[None, None, :])


def mode_face_zc(nx: int, ny: int, nz: int, p: int, q: int, r: int) -> np.ndarray:
    """Separable mode sin(p pi (i+1/2)/nx) sin(q pi (j+1/2)/ny) cos(r pi (k+1/2)/nz),
    z-contiguous (ny, nx, nz), (i, j) 0-based: the sine vanishes on the boundary faces
    (the cell-centred modes of the face-Dirichlet reading [R25])."""
    si = np.sin(p * np.pi * (np.arange(nx) + 0.5) / nx)
    sj = np.sin(q * np.pi * (np.arange(ny) + 0.5) / ny)
    ck = np.cos(r * np.pi * (np.arange(nz) + 0.5) / nz)
    return np.ascontiguousarray(sj[:, None, None] * si[None, :, None] * ck[None, None, :])


def vertical_profiles(nz: int, seed: int = 0, coupling: float = 1.0):
    """Seeded synthetic vertical profiles (a, b, c, d) of eqn:LocalMatrixStencil for a
    non-uniform column (a stretched vertical grid / varying lambda and density): positive
    interface couplings w_{k+1/2} in [0.25, 4] x `coupling` give b_k = -w_{k-1/2},
    c_k = -w_{k+1/2} (zero at the ends: Neumann), a_k, d_k in [0.5, 2].  Pure input
    generation (a splitmix64 stream), no solver arithmetic."""
    u = (_mix(np.arange(4 * nz, dtype=np.uint64), seed) + 1.0) / 2.0   # [0, 1)
    w = coupling * (0.25 + 3.75 * u[:nz])          # w[k] couples k and k+1 (w[nz-1] unused)
    b = np.zeros(nz)
    c = np.zeros(nz)
    b[1:] = -w[:nz - 1]
    c[:nz - 1] = -w[:nz - 1]
    a = 0.5 + 1.5 * u[nz:2 * nz]
    d = 0.5 + 1.5 * u[2 * nz:3 * nz]
    return a, b, c, d


def horizontal_fields(nx: int, ny: int, c: float, seed: int = 0, kind: str = "random"):
    """Seeded synthetic per-column fields of eqn:LocalMatrixStencil (|T|, alpha_{T,T'}
    "different for each horizontal grid cell T"), on the finest level:
    area [ny, nx] = |T|, ax [ny, nx+1] and ay [ny+1, nx] = alpha_{T,T'} of the x- and y-faces
    (face i of row j lies between columns i-1 and i; faces 0 and nx are boundary faces).

    kind = "random": |T| in [0.5, 2], alpha = -c x [0.25, 4] independently per cell/face
    (the hardest case for the tests); "smooth": O(1) smooth variations ("geometric
    factors arising from the spherical geometry will modify this estimate by factors of
    O(1)"): |T| = 1 + 0.4 sin(2 pi x) sin(2 pi y) and alpha = -c (1 + 0.5 cos(...)) at the
    face centres.  Pure input generation, no solver arithmetic."""
    if kind == "random":
        n_a, n_x, n_y = nx * ny, (nx + 1) * ny, nx * (ny + 1)
        u = (_mix(np.arange(n_a + n_x + n_y, dtype=np.uint64), seed + 7919) + 1.0) / 2.0   # [0, 1)
        area = (0.5 + 1.5 * u[:n_a]).reshape(ny, nx)
        ax = (-c * (0.25 + 3.75 * u[n_a:n_a + n_x])).reshape(ny, nx + 1)
        ay = (-c * (0.25 + 3.75 * u[n_a + n_x:])).reshape(ny + 1, nx)
        return area, ax, ay
    if kind != "smooth":
        raise ValueError(kind)
    xc = (np.arange(nx) + 0.5) / nx
    yc = (np.arange(ny) + 0.5) / ny
    xf = np.arange(nx + 1) / nx
    yf = np.arange(ny + 1) / ny
    ph = 0.1 * seed
    area = 1.0 + 0.4 * np.sin(2 * np.pi * (yc[:, None] + ph)) * np.sin(2 * np.pi * xc[None, :])
    ax = -c * (1.0 + 0.5 * np.cos(np.pi * (xf[None, :] + yc[:, None] + ph)))
    ay = -c * (1.0 + 0.5 * np.cos(np.pi * (xc[None, :] - yf[:, None] + ph)))
    return area, ax, ay
