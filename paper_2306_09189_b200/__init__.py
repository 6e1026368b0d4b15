"""B200-native RNS-CKKS encrypted-convolution hot path (arXiv 2306.09189).

The product is libfheconv.so (CUDA kernels for sm_100a + C++ host behind the
C ABI of include/fheconv.h). This package holds its sources (csrc/), the
in-tree build (build.py) and a ctypes host API (engine.py).
"""
from .engine import CONFIGS, Ciphertext, Context, ConvLayer, FheError, InvalidArgument, Plaintext, decompose

__all__ = ["CONFIGS", "Ciphertext", "Context", "ConvLayer", "FheError", "InvalidArgument", "Plaintext",
           "decompose"]
