"""B200-native (sm_100a) hot path of the power-method truncated SVD of arXiv 2208.08410.

The product is ``libtsvd.so`` (C ABI in ``include/tsvd.h``); ``tsvd`` is its thin ctypes
binding.  See DESIGN.md.
"""
from .tsvd import *  # noqa: F401,F403
from .tsvd import TSVD, TsvdError, lib  # noqa: F401
