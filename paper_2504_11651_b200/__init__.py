"""paper_2504_11651_b200 — B200-native DFloat11 (arXiv 2504.11651) decompression library.

The product is libdf11.so (include/df11.h): a multithreaded host encoder and sm_100a CUDA decode
kernels.  ``df11`` is the thin ctypes binding with the same names as the C ABI.
"""
from . import df11  # noqa: F401
from .df11 import (BlockPlan, DeviceTensor, Df11Error, HostTensor, decompress, decompress_block,  # noqa: F401
                   decompress_host, encode, encode_group, to_device)
