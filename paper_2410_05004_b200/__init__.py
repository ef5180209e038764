"""B200-native HCache state restoration (arXiv 2410.05004).

The product is the C-ABI library ``lib/libhcache_b200.so`` (sm_100a CUDA
kernels + the native host runtime: pinned chunk store, restore engine,
planner). ``hcache`` mirrors the reference API over it; ``sharded`` runs the
head-sharded multi-GPU restore with torch.distributed for the plumbing.
"""
from . import capi  # noqa: F401

__all__ = ["capi"]
