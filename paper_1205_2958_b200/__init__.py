"""B200-native b-bit minwise hashing preprocessing (arXiv 1205.2958 hot path).

The product is ``libbbmh.so`` (CUDA sm_100a kernels + C++ host runtime behind
the reference's C ABI, ``include/bbmh.h``); :mod:`.bbmh` is a thin ctypes
mirror of that ABI.
"""
from . import bbmh  # noqa: F401
from .bbmh import BbmhError, Family, expand_file  # noqa: F401
