"""B200-native COAT hot path: FP8-DRE AdamW, MGAQ quantizers, FP8 linear.

Importing the package loads libcoat.so (sm_100a).  There is no CPU fallback.
"""
from . import _lib  # noqa: F401  (fails loudly when libcoat.so is missing)
from . import coatsim  # noqa: F401

__all__ = ["coatsim"]
