"""B200-native Moses cost-model hot path (arXiv 2201.05752).

The compute lives in ``libmoses_gpu.so`` (hand-written sm_100a CUDA: tcgen05/TMA
GEMMs, ranking, lottery mask/update, top-k, pooling, MMD) behind the C ABI in
``include/moses_gpu.h``; ``moseslab`` mirrors the reference's C++ API over it.
"""
from . import moseslab  # noqa: F401

__all__ = ["moseslab"]
