"""Tensor profiles and contiguous partitions — the merge stage's input.

API mirror of the reference ``mergesched.profiles`` (profiles.py:36-156): a model
is its gradient tensors in backprop-readiness order (index 0 = the output layer,
whose gradient is ready first); a Partition cuts that list into contiguous groups,
each group being one fused buffer that is encoded, exchanged and decoded as a unit.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Sequence, Union


@dataclass(frozen=True)
class LayerProfile:
    """One gradient tensor (profiles.py:36-51)."""

    index: int
    size: int
    compute_time: float

    def __post_init__(self):
        if self.size < 1:
            raise ValueError(f"layer {self.index}: size must be >= 1, got {self.size}")
        if self.compute_time < 0:
            raise ValueError(f"layer {self.index}: compute_time must be >= 0, got {self.compute_time}")


@dataclass(frozen=True)
class ModelProfile:
    """Ordered tensor list (profiles.py:54-90); totals recomputed from the layers."""

    name: str
    layers: tuple
    total_size: int = field(init=False)
    total_compute: float = field(init=False)

    def __post_init__(self):
        if not self.layers:
            raise ValueError("profile needs at least one layer")
        object.__setattr__(self, "layers", tuple(self.layers))
        for pos, layer in enumerate(self.layers):
            if layer.index != pos:
                raise ValueError(f"layer indices must be 0..N-1 in order, got {layer.index} at {pos}")
        object.__setattr__(self, "total_size", sum(l.size for l in self.layers))
        object.__setattr__(self, "total_compute", math.fsum(l.compute_time for l in self.layers))

    @property
    def n_tensors(self) -> int:
        return len(self.layers)

    def sizes(self) -> list[int]:
        return [l.size for l in self.layers]

    def offsets(self) -> list[int]:
        """Element offset of every tensor inside the fused (flat) gradient buffer, plus the total."""
        out, acc = [0], 0
        for l in self.layers:
            acc += l.size
            out.append(acc)
        return out

    def to_document(self) -> dict:
        return {"name": self.name, "layers": [{"size": l.size, "compute_ms": l.compute_time} for l in self.layers]}

    @classmethod
    def from_sizes(cls, name: str, sizes: Sequence[int], compute_ms: Sequence[float] | None = None) -> "ModelProfile":
        cms = list(compute_ms) if compute_ms is not None else [0.0] * len(sizes)
        return cls(name, tuple(LayerProfile(i, int(s), float(c)) for i, (s, c) in enumerate(zip(sizes, cms))))


@dataclass(frozen=True)
class Partition:
    """Contiguous grouping of ``n_tensors`` tensors (profiles.py:93-156).  A boundary b
    cuts between tensor b-1 and tensor b; () is one merged group, all N-1 cuts is
    layer-wise."""

    n_tensors: int
    boundaries: tuple

    def __post_init__(self):
        if self.n_tensors < 1:
            raise ValueError("partition needs at least one tensor")
        cuts = tuple(int(b) for b in self.boundaries)
        object.__setattr__(self, "boundaries", cuts)
        last = 0
        for b in cuts:
            if not (1 <= b <= self.n_tensors - 1):
                raise ValueError(f"boundary {b} outside [1, {self.n_tensors - 1}]")
            if b <= last:
                raise ValueError(f"boundaries must be strictly increasing, got {cuts}")
            last = b

    @property
    def y(self) -> int:
        return len(self.boundaries) + 1

    def group_ranges(self) -> list[tuple[int, int]]:
        edges = (0, *self.boundaries, self.n_tensors)
        return list(zip(edges[:-1], edges[1:]))

    def group_counts(self) -> list[int]:
        return [b - a for a, b in self.group_ranges()]

    def group_sizes(self, profile: ModelProfile) -> list[int]:
        if profile.n_tensors != self.n_tensors:
            raise ValueError(f"partition is over {self.n_tensors} tensors, profile has {profile.n_tensors}")
        off = profile.offsets()
        return [off[b] - off[a] for a, b in self.group_ranges()]

    def element_ranges(self, profile: ModelProfile) -> list[tuple[int, int]]:
        """[start, end) element slices of each group in the fused buffer (trainer.py:344-348)."""
        off = profile.offsets()
        return [(off[a], off[b]) for a, b in self.group_ranges()]

    @classmethod
    def merged(cls, n_tensors: int) -> "Partition":
        return cls(n_tensors, ())

    @classmethod
    def layer_wise(cls, n_tensors: int) -> "Partition":
        return cls(n_tensors, tuple(range(1, n_tensors)))

    @classmethod
    def from_group_counts(cls, counts: Sequence[int]) -> "Partition":
        if any(c < 1 for c in counts):
            raise ValueError(f"group counts must be >= 1, got {list(counts)}")
        cuts, acc = [], 0
        for c in list(counts)[:-1]:
            acc += c
            cuts.append(acc)
        return cls(sum(counts), tuple(cuts))


def load_profile(document: Union[str, dict]) -> ModelProfile:
    """``{"name": str, "layers": [{"size": int, "compute_ms": float}, ...]}`` (profiles.py:159-190)."""
    if isinstance(document, str):
        try:
            document = json.loads(document)
        except json.JSONDecodeError as exc:
            raise ValueError(f"profile document is not valid JSON: {exc}") from exc
    if not isinstance(document, dict):
        raise ValueError(f"profile document must be an object, got {type(document).__name__}")
    try:
        name, raw = document["name"], document["layers"]
    except KeyError as exc:
        raise ValueError(f"profile document missing key {exc}") from exc
    if not isinstance(raw, list) or not raw:
        raise ValueError("profile 'layers' must be a non-empty list")
    layers = []
    for i, entry in enumerate(raw):
        try:
            size, compute = entry["size"], entry["compute_ms"]
        except (TypeError, KeyError):
            raise ValueError(f"layer {i}: expected object with 'size' and 'compute_ms'") from None
        if not isinstance(size, int) or isinstance(size, bool):
            raise ValueError(f"layer {i}: size must be an integer, got {size!r}")
        layers.append(LayerProfile(i, size, float(compute)))
    return ModelProfile(str(name), tuple(layers))
