"""B200-native hot path of GSCL (Bianco & Varetto, arXiv 1207.1746).

The compute lives in ``libgscl.so`` (CUDA for sm_100a behind the C ABI in
``include/gscl.h``); ``gscl`` is its ctypes binding.  Build with
``python -m paper_1207_1746_b200.build``.
"""
from . import gscl  # noqa: F401  (raises ImportError when libgscl.so is missing)

__all__ = ["gscl"]
