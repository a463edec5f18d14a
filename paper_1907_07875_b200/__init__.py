"""B200-native fast graph Fourier transform (Lu & Ortega, arXiv 1907.07875).

The product is the C-ABI library include/gft.h (libgft.so: host planner + per-plan
sm_100a kernels); `gft` is its thin ctypes binding.
"""
from .gft import *  # noqa: F401,F403
from .gft import Plan, GFTError, lib  # noqa: F401
