"""B200-native edgeset.apply (GraphIt, arXiv 1805.00923): pull / push / hybrid
edge traversal for fixed-iteration PageRank and direction-optimising BFS.

The product is the C-ABI CUDA library `libgi.so` (include/gi.h); `gi` is its
thin ctypes binding. Importing `gi` fails loudly if the library is not built.
"""
__all__ = ["gi"]
