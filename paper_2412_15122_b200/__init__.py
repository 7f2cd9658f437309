"""paper_2412_15122_b200 — B200-native warm-start APSP (arXiv 2412.15122).

The product is the C-ABI CUDA library libapsp_warm.so (include/apsp_warm.h);
``_lib`` binds it with ctypes under the same function names and ``api``
wraps it for torch tensors.  Importing this package fails if the library has
not been built — there is no CPU fallback.
"""
from . import _lib  # noqa: F401  (raises ImportError if libapsp_warm.so is missing)
from ._lib import APSP_F32, APSP_I32, APSP_INF_I32, ApspError, UpdateInfo  # noqa: F401
from .api import WarmAPSP  # noqa: F401

__all__ = ["WarmAPSP", "ApspError", "UpdateInfo", "APSP_I32", "APSP_F32", "APSP_INF_I32"]
