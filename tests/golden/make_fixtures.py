"""Record the reference fixture tensor lists (mergesched.fixtures, fixtures/__init__.py:43-102)
into tests/golden/fixtures.npz.  Run in the build container where /root/reference exists."""

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")

from mergesched.fixtures import load_fixture_profile  # noqa: E402

np.savez_compressed(
    HERE / "fixtures.npz",
    **{name: np.array([l.size for l in load_fixture_profile(name).layers], np.int64)
       for name in ("resnet50_161", "resnet101_314")},
)
print("wrote", HERE / "fixtures.npz")
