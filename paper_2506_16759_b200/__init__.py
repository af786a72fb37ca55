"""B200-native (sm_100a) bottom-up adaptive-sketching H^2 construction (arXiv 2506.16759).

The product path is libh2.so (include/h2.h); this package is its thin Python binding.
Importing it without the built library raises ImportError (no CPU fallback).
"""
from .h2 import Tree, H2Matrix, build, dense_sketch, dense_op_sketch, omega, build_opts, device_view  # noqa: F401
from ._lib import H2Error, LIB_PATH, SIGNATURES  # noqa: F401
