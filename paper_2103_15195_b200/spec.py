"""Codec configuration: the reference ``CompressorSpec`` (compressors.py:58-133)
plus its lowering to the C-ABI ``mc_spec`` struct (include/mergecomp.h)."""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

ALGORITHMS = (
    "identity", "fp16", "topk", "randk", "dgc_lite", "threshold", "qsgd",
    "signsgd", "efsignsgd", "onebit", "signum", "terngrad", "int8",
)  # wire ids = position (compressors.py:29-45)
ALGO_ID = {name: i for i, name in enumerate(ALGORITHMS)}

EF_DEFAULT_ON = frozenset({"topk", "dgc_lite", "efsignsgd", "onebit"})
SPARSIFIERS = frozenset({"topk", "randk", "dgc_lite", "threshold"})
STOCHASTIC = frozenset({"randk", "qsgd", "terngrad"})
HEADER_BYTES = 22  # canonical "<BBQIII" header (compressors.py:53)
FLAG_UNBIASED = 0x01


@dataclass(frozen=True)
class CompressorSpec:
    """One codec's configuration; fields, defaults and validation as the
    reference (compressors.py:58-92)."""

    algorithm: str
    sparsity: float = 0.99
    levels: int = 256
    bucket_size: int = 512
    error_feedback: Optional[bool] = None
    unbiased_scaling: bool = False
    threshold: float = 1e-3
    momentum: Optional[float] = None

    def __post_init__(self):
        if self.algorithm not in ALGO_ID:
            raise ValueError(f"unknown algorithm {self.algorithm!r}")
        if not (0.0 <= self.sparsity < 1.0):
            raise ValueError(f"sparsity must be in [0, 1), got {self.sparsity}")
        if self.levels < 2:
            raise ValueError(f"levels must be >= 2, got {self.levels}")
        if self.bucket_size < 1:
            raise ValueError(f"bucket_size must be >= 1, got {self.bucket_size}")
        if self.threshold < 0:
            raise ValueError(f"threshold must be >= 0, got {self.threshold}")
        if self.momentum is not None and not (0.0 <= self.momentum < 1.0):
            raise ValueError(f"momentum must be in [0, 1), got {self.momentum}")

    @property
    def uses_error_feedback(self) -> bool:
        if self.error_feedback is not None:
            return bool(self.error_feedback)
        return self.algorithm in EF_DEFAULT_ON

    @property
    def momentum_coef(self) -> Optional[float]:
        if self.algorithm == "signum":
            return 0.9 if self.momentum is None else self.momentum
        if self.algorithm == "dgc_lite" and self.momentum is not None:
            return self.momentum
        return None

    @property
    def is_stochastic(self) -> bool:
        return self.algorithm in STOCHASTIC

    @property
    def is_sparse(self) -> bool:
        return self.algorithm in SPARSIFIERS

    def to_dict(self) -> dict:
        return {
            "algorithm": self.algorithm,
            "sparsity": self.sparsity,
            "levels": self.levels,
            "bucket_size": self.bucket_size,
            "error_feedback": self.error_feedback,
            "unbiased_scaling": self.unbiased_scaling,
            "threshold": self.threshold,
            "momentum": self.momentum,
        }

    @classmethod
    def from_dict(cls, doc: dict) -> "CompressorSpec":
        if "algorithm" not in doc:
            raise ValueError("compressor spec document missing 'algorithm'")
        unknown = set(doc) - set(cls.__dataclass_fields__)
        if unknown:
            raise ValueError(f"unknown compressor spec fields: {sorted(unknown)}")
        return cls(**doc)

    def to_c(self) -> "McSpec":
        """Resolved C struct: defaults folded in (EF flag, momentum coefficient)."""
        coef = self.momentum_coef
        return McSpec(
            algorithm=ALGO_ID[self.algorithm],
            levels=int(self.levels),
            bucket_size=int(self.bucket_size),
            sparsity=float(self.sparsity),
            threshold=float(self.threshold),
            error_feedback=int(self.uses_error_feedback),
            unbiased_scaling=int(bool(self.unbiased_scaling)),
            has_momentum=int(coef is not None),
            momentum=float(coef) if coef is not None else 0.0,
        )


class McSpec(ctypes.Structure):
    """Mirror of ``mc_spec`` in include/mergecomp.h (field order matters)."""

    _fields_ = [
        ("algorithm", ctypes.c_int32),
        ("levels", ctypes.c_int32),
        ("bucket_size", ctypes.c_int64),
        ("sparsity", ctypes.c_double),
        ("threshold", ctypes.c_double),
        ("error_feedback", ctypes.c_int32),
        ("unbiased_scaling", ctypes.c_int32),
        ("has_momentum", ctypes.c_int32),
        ("momentum", ctypes.c_float),
    ]


def top_k_count(sparsity: float, length: int) -> int:
    """max(1, ceil(round((1 - sparsity) * length, 9))) — compressors.py:185-194."""
    if length < 1:
        raise ValueError("length must be >= 1")
    return max(1, math.ceil(round((1.0 - sparsity) * length, 9)))


def bucket_count(n: int, bucket_size: int) -> int:
    return (n + bucket_size - 1) // bucket_size


def level_bits(levels: int) -> int:
    return max(1, (levels - 1).bit_length())


def sign_bytes(n: int) -> int:
    return (n + 7) // 8


def code_bytes(n: int, bits_per: int) -> int:
    return (n * bits_per + 7) // 8


def section_lengths(spec: CompressorSpec, n: int, count: Optional[int] = None) -> tuple[int, int, int]:
    """(n_idx, n_val, n_bits) of the payload of an n-element group.  ``count``
    is the selected count of a threshold payload (data dependent)."""
    a = spec.algorithm
    nb = bucket_count(n, spec.bucket_size)
    if a in ("topk", "randk", "dgc_lite"):
        k = top_k_count(spec.sparsity, n)
        return k, k, 0
    if a == "threshold":
        k = top_k_count(spec.sparsity, n) if count is None else int(count)
        return k, k, 0
    if a == "identity":
        return 0, n, 0
    if a == "fp16":
        return 0, 0, 2 * n
    if a == "qsgd":
        return 0, nb, sign_bytes(n) + code_bytes(n, level_bits(spec.levels))
    if a in ("signsgd", "signum"):
        return 0, 1, sign_bytes(n)
    if a == "efsignsgd":
        return 0, nb, sign_bytes(n)
    if a == "onebit":
        return 0, 2 * nb, sign_bytes(n)
    if a == "terngrad":
        return 0, nb, code_bytes(n, 2)
    if a == "int8":
        return 0, nb, n
    raise AssertionError(a)


def payload_bytes(spec: CompressorSpec, group_size: int) -> int:
    """Canonical serialized payload size incl. the 22-byte header
    (compressors.py:565-596; threshold planned at the configured sparsity)."""
    if group_size < 1:
        raise ValueError("group_size must be >= 1")
    ni, nv, nbits = section_lengths(spec, group_size)
    return HEADER_BYTES + 4 * ni + 4 * nv + nbits
