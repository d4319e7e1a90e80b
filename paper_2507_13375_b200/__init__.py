"""B200-native GAP-LA layer-assignment hot path (arXiv 2507.13375).

``la`` is the ctypes binding of include/la.h over lib/libgapla.so (CUDA, sm_100a).
"""
__all__ = ["la"]
