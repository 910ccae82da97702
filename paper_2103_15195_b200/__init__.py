"""B200-native MergeComp compressed gradient synchronisation.

Drop-in for the reference ``mergesched`` codec / scheduler API on the
data-parallel gradient-sync path; every codec runs as hand-written sm_100a CUDA
(libmergecomp.so, C ABI in include/mergecomp.h).
"""

__version__ = "0.1.0"

from .spec import ALGORITHMS, CompressorSpec, payload_bytes, top_k_count  # noqa: F401
from .profiles import LayerProfile, ModelProfile, Partition  # noqa: F401


# The reference package root re-exports (mergesched/__init__.py:20-43), resolved lazily so
# importing the package stays cheap.  TrainConfig / TrainReport belong to the reference's
# convergence trainer (trainer.py:47-229), which is out of scope.
_LAZY = {
    "CompressedPayload": "compressors", "ResidualState": "compressors",
    "CostParams": "costmodel", "TimingSample": "costmodel",
    "SimConfig": "simulator", "SimReport": "simulator",
    "SearchConfig": "scheduler", "SearchResult": "scheduler",
}

__all__ = ["__version__", "ALGORITHMS", "CompressorSpec", "payload_bytes", "top_k_count", "LayerProfile",
           "ModelProfile", "Partition", *_LAZY]


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)
