"""REFT snapshot-and-protect, B200-native (arXiv 2310.12670).

The product is the C-ABI library ``libreft_ckpt.so`` (include/ckpt.h, CUDA sm_100a);
``paper_2310_12670_b200.ckpt`` is its thin ctypes binding (same names).  Build with
``paper_2310_12670_b200.build.build()`` (or ``__graft_entry__.build()``).
"""
from . import ckpt  # noqa: F401

__all__ = ["ckpt"]
