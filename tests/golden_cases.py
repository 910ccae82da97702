"""Loader for tests/golden/codecs.npz (reference outputs, see make_golden.py)."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from inputs import case_inputs, x_digest

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=1)
def store():
    return np.load(GOLDEN / "codecs.npz")


@lru_cache(maxsize=1)
def cases():
    return json.loads((GOLDEN / "codecs.json").read_text())["cases"]


def case_ids():
    return [c["cid"] for c in cases()]


def get_case(cid):
    for c in cases():
        if c["cid"] == cid:
            return c
    raise KeyError(cid)


def inputs(c):
    z = store()
    xs = case_inputs(c)
    for t, row in enumerate(xs):
        for w, x in enumerate(row):
            key = f"{c['cid']}.t{t}.w{w}"
            assert int(z[key + ".xdigest"][0]) == x_digest(x), f"input drift in {key}"
    return xs


def field(cid, t, w, name):
    z = store()
    key = f"{cid}.t{t}.w{w}.{name}"
    return z[key] if key in z.files else None


def mean(cid, t):
    return store()[f"{cid}.t{t}.mean"]


def seed(cid, t, w):
    s = store()[f"{cid}.t{t}.w{w}.seed"]
    return int(s[0]) | (int(s[1]) << 64)
