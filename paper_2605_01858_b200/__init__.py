"""B200-native (sm_100a) DSCache streaming KV-cache hot path.

The product is the C-ABI library ``libdscache.so`` (include/dscache.h);
``dscache`` is its ctypes binding.  See DESIGN.md.
"""
from .dscache import DSCache, DSCacheError, load_library  # noqa: F401

__all__ = ["DSCache", "DSCacheError", "load_library"]
