"""paper_1707_02000_b200 — B200-native (sm_100a) PKT truss decomposition.

The product is lib/libtdg.so (CUDA kernels + the C-ABI of include/tdg.h). This package
adds the host mirrors of the reference interface: ``trussdec`` (Python, ctypes) and
``shim/trussdec_gpu.hpp`` (C++). ``graphgen`` is the seeded config generator used by the
benchmark and tests.
"""
from ._lib import build, ensure_built, TdgError  # noqa: F401

__all__ = ["build", "ensure_built", "TdgError"]
