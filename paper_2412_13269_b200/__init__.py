"""B200-native drop-in for the RNS-CKKS evaluation path of TETRIS
(arXiv 2412.13269): NTT, element-wise modular arithmetic, hybrid key switching,
Galois rotations, Chebyshev / minimax-sign evaluation and slot sums, as
hand-written sm_100a CUDA kernels behind the C-ABI in include/tetris_b200.h,
with the reference's C++ API (include/tetris_b200/*.hpp) on top.

`paper_2412_13269_b200.tetris` is the Python binding of that C++ API. There is
no CPU fallback: importing fails loudly if the extension is not built, and
every arithmetic call raises TetrisError("[gpu] ...") without a CUDA device.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libtetris_b200.so"
HEADER_PATH = _PKG.parent / "include" / "tetris_b200.h"

try:
    from . import _tetris_b200 as tetris  # noqa: F401  (the C++ API binding)
except ImportError as e:  # pragma: no cover - exercised only on a broken build
    raise ImportError(
        "paper_2412_13269_b200: native extension not built "
        "(run `python __graft_entry__.py build`): " + str(e)) from e


def load_c_abi() -> ctypes.CDLL:
    """The C-ABI shared library (include/tetris_b200.h) for ctypes callers."""
    return ctypes.CDLL(str(LIB_PATH))


__all__ = ["tetris", "load_c_abi", "LIB_PATH", "HEADER_PATH"]
