"""Stage the reference package into ``oracle/_ref/pkg`` — TEST INFRASTRUCTURE ONLY.

The reference (``/root/reference/pkg``: the ``mergesched`` package and its pytest
suite) is pure Python/numpy: there is nothing to compile, so the "build" of
``oracle/_ref`` is an unmodified copy of ``pkg/src/mergesched``, ``pkg/tests`` and
``pkg/pyproject.toml``.  ``oracle/_ref/`` is git-ignored (never part of the
repository's history) and not gpurun-ignored, so it travels to the GPU box next to
the built ``.so`` — the box itself never reads /root/reference.

Two consumers, both test/measurement legs:

* ``tests/test_gpu_reference_suite.py`` runs the reference's own tests with
  ``mergesched.compressors`` replaced by ``paper_2103_15195_b200.compressors``
  (INTEGRATION.md §1): the drop-in proof on the B200;
* ``bench.py --impl reference`` / ``cpu_baseline`` time the reference's own
  encode/aggregate loop (``kind: "reference"``).

    python oracle/stage_ref.py [/root/reference]
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
DEST = HERE / "_ref" / "pkg"


def stage(ref_root: Path = Path("/root/reference")) -> Path | None:
    pkg = ref_root / "pkg"
    if not (pkg / "src" / "mergesched").is_dir():
        return None  # GPU box / no reference: keep whatever was staged before
    if DEST.exists():
        shutil.rmtree(DEST)
    ign = shutil.ignore_patterns("__pycache__", "*.pyc", "*.egg-info", ".pytest_cache")
    shutil.copytree(pkg / "src" / "mergesched", DEST / "src" / "mergesched", ignore=ign)
    shutil.copytree(pkg / "tests", DEST / "tests", ignore=ign)
    shutil.copy2(pkg / "pyproject.toml", DEST / "pyproject.toml")
    return DEST


def ref_src() -> Path | None:
    """Path to put on sys.path to import the staged reference, or None."""
    p = DEST / "src"
    return p if (p / "mergesched" / "compressors.py").exists() else None


if __name__ == "__main__":
    print(stage(Path(sys.argv[1]) if len(sys.argv) > 1 else Path("/root/reference")))
