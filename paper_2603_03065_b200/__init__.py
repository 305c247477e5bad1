"""B200-native fixed-shape IVF-PQ query path of V3DB (arxiv 2603.03065).

The product is libv3db.so (C ABI in include/v3db.h, CUDA kernels for sm_100a in csrc/);
``v3db`` is its thin Python binding.  See DESIGN.md.
"""
from . import _lib  # noqa: F401
