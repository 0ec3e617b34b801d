"""B200-native hot path of GSCL (Bianco & Varetto, arXiv 1207.1746).

The compute lives in ``libgscl.so`` (CUDA for sm_100a behind the C ABI in
``include/gscl.h``); ``gscl`` is its ctypes binding.  Build with
``python -m paper_1207_1746_b200.build``.

``gscl`` is imported on first access (PEP 562) so that the build module can be
imported from a fresh checkout, before ``libgscl.so`` exists.  Accessing
``paper_1207_1746_b200.gscl`` without the library raises ``ImportError``: there
is no fallback.
"""
import importlib

__all__ = ["gscl"]


def __getattr__(name):
    if name == "gscl":
        return importlib.import_module(".gscl", __name__)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
