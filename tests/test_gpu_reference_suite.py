"""The drop-in proof: the reference's OWN test suite, unmodified, with its codec module
replaced by ours (``sys.modules["mergesched.compressors"] =
paper_2103_15195_b200.compressors``), run on the B200.

The reference package and tests are staged unmodified into ``oracle/_ref/pkg`` by
``oracle/stage_ref.py`` (called from ``__graft_entry__.build()`` in the build container;
git-ignored, travels to the GPU box).  The reference's Trainer, cost model and simulator
stay the reference's code and call our codecs.  Selected suites:

* ``test_compressors.py`` — every codec's selection rules, quantizer semantics, EF
  decomposition, payload sizing, serialization (hypothesis property tests included);
* ``test_acceptance.py::test_08_compressor_suite`` — EF exactness, k-selection, the
  seed-tuned Monte-Carlo unbiasedness band (qsgd root 14, randk root 2), the
  serialize/deserialize roundtrip of all 13 codecs;
* ``test_trainer.py`` — incl. ``TestSynchrony`` (replicas bitwise identical after every
  compressed step).
"""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "oracle" / "_ref" / "pkg"

SUITES = [
    "tests/test_compressors.py",
    "tests/test_acceptance.py::test_08_compressor_suite",
    "tests/test_trainer.py",
]


@pytest.mark.skipif(not (PKG / "tests").is_dir(), reason="reference not staged (oracle/stage_ref.py)")
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_through_gpu_codecs(suite):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(PKG / "src"), str(ROOT), str(ROOT / "tests" / "refshim"),
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "mergecomp_shim", "-p", "no:cacheprovider",
           "--rootdir", str(PKG), suite]
    r = subprocess.run(cmd, cwd=PKG, env=env, capture_output=True, text=True, timeout=1800)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    m = re.search(r"MC_KERNEL_LAUNCHES=(\d+)", r.stdout)
    assert m and int(m.group(1)) > 0, "the reference suite did not run the GPU codecs\n" + tail
    print(tail)
