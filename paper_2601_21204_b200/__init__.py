"""B200-native (sm_100a) N-gram Embedding hot path (arXiv 2601.21204, LongCat-Flash-Lite).

The product is libngram_b200.so (csrc/: CUDA kernels + C++ host layer behind the C-ABI
in include/ngram_b200.h).  `abi` binds that ABI with ctypes; `ngram` mirrors the
reference's C++ API names on top of it.  There is no CPU fallback: importing `ngram`
without the built library raises.
"""
__all__ = ["abi", "ngram", "build"]
