"""B200-native (sm_100a) hot path of Asynchronous Expert Parallelism (arXiv 2505.08944).

The product is libamoe.so (csrc/, C ABI in include/amoe.h); `amoe` is its thin ctypes binding.
"""
from . import amoe  # noqa: F401
