"""hadacodec-b200: B200-native per-pixel core of Hadamard spectral codes.

The product is ``libhadacodec_b200.so`` (hand-written sm_100a CUDA behind the
C ABI in ``include/hadacodec_b200.h``); this package builds it
(:mod:`.build`), binds it (:mod:`._lib`) and mirrors the reference's host
interface over torch CUDA tensors (:mod:`.api`).  Importing the package does
not load the library; the first call does, and fails loudly if it is missing.
"""
from .colorimetry import GRIDS, cmf_matrix, grid, wavelengths  # noqa: F401

__all__ = ["GRIDS", "cmf_matrix", "grid", "wavelengths"]
__version__ = "0.1.0"
