"""B200-native binned componentwise gradient boosting (arXiv 2110.03513).

The engine is the C-ABI library libcwb.so (include/cwb.h, CUDA for sm_100a);
this package only builds it (build.py) and binds it (cwb.py).
"""
from . import cwb  # noqa: F401
from .cwb import Config, CwbError, Pool  # noqa: F401
