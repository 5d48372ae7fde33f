"""B200-native PtyGer ML-CG iteration (arXiv 2106.07575).

The compute path is libptyger.so (hand-written sm_100a CUDA behind the C ABI of
include/ptyger.h); this package is its thin ctypes binding plus the seeded input
generator (``inputs``).  Importing ``paper_2106_07575_b200.ptyger`` fails loudly when
the library is not built.
"""
__all__ = ["inputs"]


def __getattr__(name):
    if name == "ptyger":
        from . import _lib as ptyger
        return ptyger
    raise AttributeError(name)
