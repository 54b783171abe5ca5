"""B200-native register-cache stencil library (arxiv 2301.11389 hot path).

The compute path is the C-ABI shared library ``libstencil_b200.so`` built
from ``csrc/`` (hand-written sm_100a CUDA).  ``binding`` is a thin ctypes
layer over it; importing this package does not load the library, so the
input generator can be used on hosts without a GPU.
"""
__all__ = ["binding", "inputs"]
