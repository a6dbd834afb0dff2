"""B200-native Live WDD hot path (arXiv 2212.01309): C-ABI library libwdd.so + ctypes binding.

See include/wdd.h for the boundary and DESIGN.md for the design.  The oracle under oracle/
is test infrastructure and is never imported from here.
"""
from .wdd import Plan, WddError, link_shards, load_library, nccl_unique_id, LIB_PATH  # noqa: F401
