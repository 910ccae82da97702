"""Deterministic golden-case inputs (shared by make_golden.py and the tests).

Large cases are not stored in the .npz: they are regenerated here from the
case id with numpy's default_rng (same numpy in the build container and on the
GPU box) and checked against the stored crc32 digest before use.
"""

from __future__ import annotations

import zlib

import numpy as np


def _one(rng, n, style):
    x = (rng.standard_normal(n) * rng.uniform(0.5, 2.0)).astype(np.float32)
    if style == "zeros" and n >= 8:
        # an all-zero span (zero-bucket skip in qsgd/terngrad/int8) + a signed zero
        lo = n // 3
        x[lo:lo + max(1, n // 4)] = 0.0
        x[1] = -0.0
    if style == "dyadic":
        x = (rng.integers(-64, 65, size=n) * 2.0 ** -6).astype(np.float32)
    return x


def case_inputs(c: dict) -> list[list[np.ndarray]]:
    """xs[t][w] for a case dict {cid, n, workers, iters, style}."""
    rng = np.random.default_rng(sum(map(ord, c["cid"])) * 7919 + c["n"])
    out = []
    for _t in range(c["iters"]):
        row = []
        for _w in range(c["workers"]):
            x = _one(rng, c["n"], c["style"])
            if c["cid"] == "fp16_range":
                x = (np.sign(x) * np.exp2(rng.uniform(-30, 18, c["n"]))).astype(np.float32)
            row.append(x)
        out.append(row)
    return out


def x_digest(x: np.ndarray) -> int:
    return zlib.crc32(np.ascontiguousarray(x, np.float32).tobytes())
