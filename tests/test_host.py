"""CPU-only tests: the C-ABI library loads and exports every symbol the header
declares (no GPU needed), host logic of the API mirror (spec validation, sizes,
seed derivation, partitions, gradient-set shapes, scheduler) against the oracle
and the reference's documented behaviour."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import mergecomp_oracle as O
from paper_2103_15195_b200 import gradsets
from paper_2103_15195_b200.profiles import LayerProfile, ModelProfile, Partition, load_profile
from paper_2103_15195_b200.spec import ALGORITHMS, CompressorSpec, payload_bytes, top_k_count

ROOT = Path(__file__).resolve().parents[1]


# ------------------------------------------------------------------ C ABI
def _declared_symbols():
    text = (ROOT / "include" / "mergecomp.h").read_text()
    return sorted(set(re.findall(r"\b(mc_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = _declared_symbols()
    for required in ("mc_encode", "mc_decode_mean", "mc_encode_decode", "mc_payload_bytes", "mc_derive_seed",
                     "mc_pack", "mc_unpack", "mc_serialize", "mc_top_k_count"):
        assert required in syms


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2103_15195_b200 import _native

    so = _native.lib()  # raises loudly if the .so is missing
    for name in _declared_symbols():
        assert hasattr(so, name), name
    assert set(_native.EXPORTED) <= set(_declared_symbols())
    assert so.mc_abi_version() == 1


def test_native_host_functions_match_reference_semantics():
    from paper_2103_15195_b200 import _native

    so = _native.lib()
    for s, n in [(0.5, 4), (0.99, 10000), (0.99, 1), (0.7, 10), (0.0, 8), (0.999, 25_557_032), (0.95, 599)]:
        assert so.mc_top_k_count(s, n) == top_k_count(s, n) == O.keep_count(s, n)
    for algo in ALGORITHMS:
        for kw in ({}, {"levels": 16, "bucket_size": 50}, {"sparsity": 0.5}, {"levels": 5, "bucket_size": 7}):
            spec = CompressorSpec(algo, **kw)
            cs = spec.to_c()
            for n in (1, 7, 63, 512, 1000, 4109, 10 ** 6 + 3):
                assert so.mc_payload_bytes(ctypes.byref(cs), n) == payload_bytes(spec, n) == O.payload_bytes(spec, n)


def test_native_derive_seed_matches_numpy_seedsequence():
    from paper_2103_15195_b200 import _native
    from paper_2103_15195_b200._seedseq import seed_sequence_key

    for args in [(0, 0, 0, 0), (7, 1, 2, 3), (2 ** 32 + 5, 3, 999, 7), (2 ** 63 + 11, 0, 1, 1), (123, 4, 5, 6)]:
        lo, hi = _native.derive_key(*args)
        assert (lo | hi << 64) == O.derive_seed(*args)
        assert seed_sequence_key(list(args)) == (lo, hi)
    lo, hi = seed_sequence_key([2 ** 70 + 1, 2, 3, 4])  # > 64-bit entropy: Python path
    assert (lo | hi << 64) == O.derive_seed(2 ** 70 + 1, 2, 3, 4)


def test_device_layout_is_aligned_and_sized():
    from paper_2103_15195_b200 import _native

    for algo in ALGORITHMS:
        spec = CompressorSpec(algo, levels=16 if algo == "qsgd" else 256)
        for n in (1, 9, 1000, 25_557_032):
            L = _native.layout(spec.to_c(), n)
            assert L.bytes % 16 == 0 and L.off_val % 16 == 0 and L.off_bits % 16 == 0 and L.off_codes % 16 == 0
            # the device payload carries at least the canonical sections
            assert L.bytes >= payload_bytes(spec, n) - 22 + 32 - 16 or spec.is_sparse


def test_workspace_query():
    from paper_2103_15195_b200 import _native

    for algo in ALGORITHMS:
        assert _native.workspace_bytes(CompressorSpec(algo).to_c(), 12345) >= 64


# ------------------------------------------------------------------ API mirror (host)
def test_spec_validation_and_defaults():
    for kw in ({"sparsity": 1.0}, {"sparsity": -0.1}, {"levels": 1}, {"bucket_size": 0}, {"threshold": -1.0},
               {"momentum": 1.0}):
        with pytest.raises(ValueError):
            CompressorSpec("topk", **kw)
    with pytest.raises(ValueError):
        CompressorSpec("gzip")
    assert CompressorSpec("efsignsgd").uses_error_feedback and not CompressorSpec("qsgd").uses_error_feedback
    assert CompressorSpec("signum").momentum_coef == 0.9 and CompressorSpec("dgc_lite").momentum_coef is None
    spec = CompressorSpec("qsgd", levels=16, bucket_size=64, error_feedback=True)
    assert CompressorSpec.from_dict(spec.to_dict()) == spec
    with pytest.raises(ValueError):
        CompressorSpec.from_dict({"algorithm": "topk", "ratio": 0.5})


def test_partitions():
    p = Partition(10, (3, 7))
    assert p.y == 3 and p.group_ranges() == [(0, 3), (3, 7), (7, 10)] and p.group_counts() == [3, 4, 3]
    assert Partition.from_group_counts([2, 2]).boundaries == (2,)
    assert Partition.layer_wise(4).boundaries == (1, 2, 3) and Partition.merged(4).y == 1
    for bad in [(0,), (10,), (3, 3), (5, 2)]:
        with pytest.raises(ValueError):
            Partition(10, bad)
    prof = ModelProfile.from_sizes("m", [5, 6, 7, 8])
    assert Partition(4, (1, 3)).group_sizes(prof) == [5, 13, 8]
    assert Partition(4, (1, 3)).element_ranges(prof) == [(0, 5), (5, 18), (18, 26)]
    doc = prof.to_document()
    assert load_profile(doc) == prof
    with pytest.raises(ValueError):
        load_profile('{"name": "x", "layers": []}')
    with pytest.raises(ValueError):
        ModelProfile("x", (LayerProfile(1, 3, 0.0),))


def test_gradient_sets_match_reference_shapes():
    z = np.load(ROOT / "tests" / "golden" / "fixtures.npz")
    for name in ("resnet50_161", "resnet101_314"):
        assert list(gradsets.sizes(name)) == z[name].tolist()
    assert (len(gradsets.sizes("resnet50_161")), sum(gradsets.sizes("resnet50_161"))) == (161, 25_557_032)
    assert (len(gradsets.sizes("resnet101_314")), sum(gradsets.sizes("resnet101_314"))) == (314, 44_549_160)
    assert (len(gradsets.sizes("maskrcnn_201")), sum(gradsets.sizes("maskrcnn_201"))) == (201, 44_454_513)
    assert (len(gradsets.sizes("vgg16_32")), sum(gradsets.sizes("vgg16_32"))) == (32, 138_357_544)
    g = gradsets.synthetic_gradients("tiny40", 1, 0)
    assert g.dtype == np.float32 and g.size == sum(gradsets.sizes("tiny40"))


# ------------------------------------------------------------------ scheduler (host logic)
def _quadratic_evaluator(profile, best):
    return lambda part: (sum((b - c) ** 2 for b, c in zip(part.boundaries, best)) + 1.0) * (1 + 0.01 * part.y)


def test_heuristic_search_finds_planted_split():
    from paper_2103_15195_b200.scheduler import SearchConfig, heuristic_search, optimal_split_y2

    prof = ModelProfile.from_sizes("m", [10] * 161)
    f = lambda part: 5.0 if part.y == 1 else 1.0 + (part.boundaries[0] - 120) ** 2 * 1e-3  # noqa: E731
    j, v = optimal_split_y2(f, prof)
    assert j == 120 and v == 1.0
    res = heuristic_search(SearchConfig(Y=2, evaluator=f), prof)
    assert res.partition.boundaries == (120,) and res.termination == "reached_Y" and res.evaluations < 50


def test_search_stops_when_more_groups_are_worse():
    from paper_2103_15195_b200.scheduler import SearchConfig, heuristic_search

    prof = ModelProfile.from_sizes("m", [10] * 30)
    res = heuristic_search(SearchConfig(Y=3, evaluator=lambda p: 1.0 + p.y), prof)
    assert res.partition.y == 1 and res.termination == "worse_than_prev"
    res = heuristic_search(SearchConfig(Y=3, alpha=0.5, evaluator=lambda p: 2.0 - 0.1 * (p.y > 1)), prof)
    assert res.termination == "marginal_benefit" and res.partition.y == 2


def test_online_search_pins_and_uses_median():
    from paper_2103_15195_b200.scheduler import SearchConfig, measured_evaluator, online_search

    class Handle:
        def __init__(self):
            self.calls, self.pinned = 0, None

        def tensor_profile(self):
            return ModelProfile.from_sizes("m", [4] * 20)

        def timed_iteration(self, part):
            self.calls += 1
            jitter = 100.0 if self.calls % 5 == 0 else 0.0  # outliers must not move the median
            return 1.0 + (0 if part.y == 1 else abs(part.boundaries[0] - 7)) * 0.1 + jitter - (part.y > 1) * 0.5

        def pin_partition(self, part):
            self.pinned = part

    h = Handle()
    res = online_search(SearchConfig(Y=2), h, repetitions=5)
    assert h.pinned == res.partition and res.partition.boundaries == (7,)
    with pytest.raises(ValueError):
        measured_evaluator(h, 0)


def test_exhaustive_matches_heuristic_on_unimodal():
    from paper_2103_15195_b200.scheduler import SearchConfig, exhaustive_search, heuristic_search, naive_partition

    prof = ModelProfile.from_sizes("m", [3] * 12)
    f = lambda p: 10.0 if p.y == 1 else (1.0 + (p.boundaries[0] - 4) ** 2 if p.y == 2 else 50.0)  # noqa: E731
    ex = exhaustive_search(f, prof, y_max=2)
    he = heuristic_search(SearchConfig(Y=2, evaluator=f), prof)
    assert ex.partition == he.partition == Partition(12, (4,))
    assert naive_partition(prof, 5).group_counts() == [3, 3, 2, 2, 2]


def test_package_root_reexports_reference_names():
    """mergesched/__init__.py:20-43 re-exports, minus the out-of-scope trainer types."""
    import paper_2103_15195_b200 as P

    for name in ("LayerProfile", "ModelProfile", "Partition", "CompressorSpec", "CompressedPayload",
                 "ResidualState", "CostParams", "TimingSample", "SimConfig", "SimReport", "SearchConfig",
                 "SearchResult"):
        assert getattr(P, name).__name__ == name
        assert name in P.__all__


def test_bench_cli_parses():
    """bench.py (the driver's entry) parses and prints its usage without a GPU."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--help"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "--e2e-chunk" in r.stdout


def test_chunk_ranges_cover_group_on_bucket_and_word_boundaries():
    """GradSync's N > 1 chunk pipeline: chunks tile the group exactly, every chunk but the
    last is a multiple of lcm(bucket_size, 32) (so chunk-wise encodes equal the whole-group
    encode), automatic only for the byte codecs and only for groups >= 2 CHUNK_MIN."""
    import math
    from types import SimpleNamespace

    from paper_2103_15195_b200.spec import CompressorSpec
    from paper_2103_15195_b200.sync import GradSync

    def ranges(algo, n, world=2, chunk=None, bucket=512):
        obj = SimpleNamespace(world=world, chunk_elems=chunk, spec=CompressorSpec(algo, bucket_size=bucket),
                              CHUNKABLE=GradSync.CHUNKABLE, CHUNK_AUTO=GradSync.CHUNK_AUTO,
                              CHUNK_MIN=GradSync.CHUNK_MIN)
        return GradSync._chunk_ranges(obj, n)

    assert ranges("int8", 25_557_032, world=1) is None               # one rank: nothing to overlap
    assert ranges("efsignsgd", 25_557_032) is None                   # 1-bit codecs: not by default
    assert ranges("qsgd", 25_557_032, chunk=1 << 20) is None         # stream offsets span the group
    assert ranges("int8", 3_000_000) is None                         # small group
    for algo, n, chunk, bucket in [("int8", 25_557_032, None, 512), ("fp16", 44_555_013, None, 512),
                                   ("efsignsgd", 100_003, 1024, 512), ("onebit", 100_003, 1000, 50)]:
        r = ranges(algo, n, chunk=chunk, bucket=bucket)
        assert r is not None and r[0][0] == 0 and r[-1][1] == n
        align = bucket * 32 // math.gcd(bucket, 32)
        for (a, b), (c, _) in zip(r, r[1:]):
            assert b == c and (b - a) % align == 0
