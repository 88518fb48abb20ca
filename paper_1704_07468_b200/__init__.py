"""B200-native gapped k-mer kernel matrices by sort-and-count (GaKCo, arXiv 1704.07468).

The compute path is libgakco.so (CUDA, sm_100a) behind the C-ABI in include/gakco.h;
`gakco` is its ctypes binding. See DESIGN.md.
"""
from . import gakco  # noqa: F401
from .gakco import Plan, kernel_matrix  # noqa: F401
