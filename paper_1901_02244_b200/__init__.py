"""B200-native hot path of Synchronous Model Averaging (SMA), arXiv 1901.02244.

``libsma.so`` (CUDA C++ for sm_100a behind the C ABI in ``include/sma.h``) does
all the arithmetic; ``paper_1901_02244_b200.sma`` is the ctypes binding.
"""
from . import sma  # noqa: F401
from .sma import Sma, SmaError  # noqa: F401
