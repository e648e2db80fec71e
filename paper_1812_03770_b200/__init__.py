"""B200-native evaluator for Owl-style computation graphs (arXiv 1812.03770).

The product is libcg.so (include/cg.h): host compiler (C++), NVRTC-generated
sm_100a group kernels and hand-written kernels.  ``cg`` is its ctypes binding.
"""
from . import cg  # noqa: F401
