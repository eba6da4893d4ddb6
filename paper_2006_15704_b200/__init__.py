"""B200-native DDP Reducer gradient synchronization (arXiv 2006.15704).

Native library: ``lib/libb200ddp.so`` (C ABI: ``include/b200ddp.h``).
``_lib``: ctypes binding (same names as the C ABI).  ``ddp``: thin PyTorch
front end (hooks, symmetric memory, process-group bootstrap).
"""

__all__ = ["_lib", "ddp"]
