"""B200-native in situ Lagrangian flow-map extraction (arXiv 2004.02003).

The product is liblag.so (C ABI, include/lag.h) built from the sm_100a CUDA
kernels in csrc/.  This package is the thin Python binding over it.  Inputs
come from the separate `lag_inputs` package; the CPU oracle (`oracle/`) is
test infrastructure and is never imported here.
"""
from .lag import *  # noqa: F401,F403
from .lag import Context, LagError, load, make_config, EXPORTS, LIB_PATH  # noqa: F401
