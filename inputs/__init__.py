"""Seeded synthetic inputs shared by the oracle side (tests) and the GPU side.

This module holds none of the method's arithmetic: only the counter-based
random generator for the right-hand side (splitmix64 keyed by the global
Lambda index) and the separable Fourier modes
used to build manufactured fields.  Both the numpy version here and the CUDA
version in ``splitmix_gpu.cu`` produce bit-identical values.
"""
from .splitmix import rhs_lambda, rhs_zc, mode_zc, mode_face_zc, vertical_profiles, horizontal_fields, GOLDEN  # noqa: F401
