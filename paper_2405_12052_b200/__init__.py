"""B200-native Lloyd's K-means iteration (arXiv 2405.12052).

The compute path is the C-ABI library ``libkmeans.so`` (hand-written sm_100a
CUDA, see ``include/kmeans.h``); ``paper_2405_12052_b200.kmeans`` is its thin
ctypes binding.  ``datagen`` holds the seeded synthetic input recipe.

Importing this package does not load the CUDA library; ``kmeans`` does, and
raises if the extension has not been built (there is no CPU fallback).
"""
__all__ = ["datagen", "kmeans"]
