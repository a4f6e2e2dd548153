"""B200-native MTI-pruned Lloyd's k-means (arXiv 1902.09527, clusterNOR/knor hot path).

The product is ``libkmeans_b200.so`` (hand-written sm_100a CUDA + a C ABI, see
``include/kmeans_b200.h``); this package is its thin Python binding.
"""
from .kmeans import KMeans, default_options, kmeanspp_multirun, nccl_unique_id, seed_plusplus  # noqa: F401
from ._capi import KMeansError, SO_PATH  # noqa: F401

__version__ = "0.1.0"
