"""B200-native MergeComp compressed gradient synchronisation.

Drop-in for the reference ``mergesched`` codec / scheduler API on the
data-parallel gradient-sync path; every codec runs as hand-written sm_100a CUDA
(libmergecomp.so, C ABI in include/mergecomp.h).
"""

__version__ = "0.1.0"

from .spec import ALGORITHMS, CompressorSpec, payload_bytes, top_k_count  # noqa: F401
from .profiles import LayerProfile, ModelProfile, Partition  # noqa: F401


def __getattr__(name):  # lazy: importing the package never needs a GPU
    if name in ("CompressedPayload", "ResidualState"):
        from . import compressors

        return getattr(compressors, name)
    if name in ("SearchConfig", "SearchResult"):
        from . import scheduler

        return getattr(scheduler, name)
    raise AttributeError(name)
