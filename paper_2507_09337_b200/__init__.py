"""B200-native (sm_100a, fp64) hot path of ORCHA's Flash-X Sedov case study
(arXiv 2507.09337): the per-block explicit hydro update of a packet of N
equal blocks with guard cells, behind the C ABI of include/orcha.h.

    liborcha.so         production build (FMA)      -- abi.load(False)
    liborcha_parity.so  parity build (--fmad=false) -- abi.load(True)

This package never imports the CPU oracle (oracle/) and has no CPU path.
"""
from . import abi  # noqa: F401

__all__ = ["abi"]
