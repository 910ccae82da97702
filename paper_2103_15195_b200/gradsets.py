"""Synthetic gradient sets of the BASELINE.json configs.

* resnet50_161 / resnet101_314 — the reference fixture tensor lists
  (fixtures/__init__.py:43-102): bottleneck ResNets, backprop order, sizes only.
* maskrcnn_201 / vgg16_32 — torchvision model tensor lists (data/gradsets.json,
  written by scripts/make_gradsets.py).

Values: per-tensor N(0, sigma_t^2) float32 with sigma_t log-uniform in [1e-5, 1e-2],
drawn from numpy default_rng(1000 * iteration + rank) so the host oracle sees the
same bits; one tensor per set is all zeros (exercises the zero-bucket skip).
"""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from .profiles import ModelProfile

DATA = Path(__file__).resolve().parent / "data" / "gradsets.json"


def _bottleneck_resnet(blocks: tuple[int, ...]) -> list[int]:
    """Forward-order parameter sizes of a torchvision-style bottleneck ResNet."""
    fwd = [64 * 3 * 7 * 7, 64, 64]  # stem conv + bn
    cin = 64
    for stage, nblk in enumerate(blocks):
        width = 64 << stage
        cout = 4 * width
        for b in range(nblk):
            fwd += [width * cin, width, width,             # 1x1 reduce + bn
                    width * width * 9, width, width,       # 3x3 + bn
                    cout * width, cout, cout]              # 1x1 expand + bn
            if b == 0:
                fwd += [cout * cin, cout, cout]            # projection shortcut + bn
            cin = cout
    fwd += [2048 * 1000, 1000]  # fc
    return fwd


@lru_cache(maxsize=None)
def sizes(name: str) -> tuple[int, ...]:
    """Backprop-ordered tensor sizes of a named gradient set."""
    if name == "resnet50_161":
        return tuple(reversed(_bottleneck_resnet((3, 4, 6, 3))))
    if name == "resnet101_314":
        return tuple(reversed(_bottleneck_resnet((3, 4, 23, 3))))
    doc = json.loads(DATA.read_text())
    if name in doc:
        return tuple(doc[name])
    if name.startswith("tiny"):  # small set for tests / smoke: tiny<N>
        n = int(name[4:] or 24)
        rng = np.random.default_rng(n)
        return tuple(int(v) for v in rng.integers(1, 5000, size=n))
    raise KeyError(f"unknown gradient set {name!r}")


def profile(name: str) -> ModelProfile:
    return ModelProfile.from_sizes(name, sizes(name))


def synthetic_gradients(name: str, iteration: int = 0, rank: int = 0, zero_tensor: int = 1) -> np.ndarray:
    """Flat float32 gradient buffer (backprop order) for one (iteration, rank)."""
    sz = sizes(name)
    rng = np.random.default_rng(1000 * iteration + rank)
    sig = np.exp(rng.uniform(np.log(1e-5), np.log(1e-2), size=len(sz)))
    out = np.empty(sum(sz), np.float32)
    off = 0
    for t, (s, sd) in enumerate(zip(sz, sig)):
        if t == zero_tensor:
            out[off:off + s] = 0.0
        else:
            out[off:off + s] = rng.standard_normal(s, dtype=np.float32) * np.float32(sd)
        off += s
    return out
