"""Pin the CPU oracle to the reference: every golden vector recorded from the
real ``mergesched`` package (tests/golden/make_golden.py) must be reproduced
bit for bit by oracle/mergecomp_oracle.py.  CPU only."""

import numpy as np
import pytest

import golden_cases as G
import mergecomp_oracle as O
from paper_2103_15195_b200.spec import CompressorSpec

TIE_CASES = {"topk_dyadic_ef"}  # dyadic grid: ties at the k-th magnitude are expected


def _bits_equal(a, b):
    if a is None or b is None:
        return (a is None or len(a) == 0) and (b is None or len(b) == 0)
    return a.dtype == b.dtype and a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("cid", G.case_ids())
def test_oracle_reproduces_reference(cid):
    c = G.get_case(cid)
    spec = CompressorSpec(**c["spec"])
    xs = G.inputs(c)
    states = [None] * c["workers"]
    for t in range(c["iters"]):
        seeds = [G.seed(cid, t, w) for w in range(c["workers"])]
        assert seeds == [O.derive_seed(c["root"], w, t, 0) for w in range(c["workers"])]
        mean, payloads, states = O.sync_group(spec, xs[t], states, seeds)
        for w, p in enumerate(payloads):
            if cid in TIE_CASES:
                # tie contract: same count; EF decomposition exact
                assert len(p.indices) == len(G.field(cid, t, w, "idx"))
                continue
            assert _bits_equal(p.indices, G.field(cid, t, w, "idx")), (cid, t, w, "idx")
            assert _bits_equal(p.values, G.field(cid, t, w, "val")), (cid, t, w, "val")
            assert _bits_equal(p.bits, G.field(cid, t, w, "bits")), (cid, t, w, "bits")
            assert p.flags == int(G.field(cid, t, w, "flags")[0])
            ser = G.field(cid, t, w, "ser")
            if ser is not None:
                assert O.serialize(p) == ser.tobytes()
                assert p.byte_size == len(ser)
            dec = G.field(cid, t, w, "dec")
            if dec is not None:
                assert _bits_equal(O.decode(spec, p), dec)
            res = G.field(cid, t, w, "res")
            if res is not None:
                assert _bits_equal(states[w].residual, res), (cid, t, w, "res")
            mom = G.field(cid, t, w, "mom")
            if mom is not None:
                assert _bits_equal(states[w].momentum, mom), (cid, t, w, "mom")
        if cid not in TIE_CASES:
            assert _bits_equal(mean, G.mean(cid, t)), (cid, t, "mean")


def test_derive_seed_table():
    for root, w, t, g, lo, hi in G.store()["derive_seed.table"].tolist():
        assert O.derive_seed(root, w, t, g) == (lo | (hi << 64))


@pytest.mark.parametrize("n", [int(v) for v in G.store()["mean.lengths"]])
def test_pairwise_mean_restatement(n):
    z = G.store()
    a = z[f"mean.n{n}.a"]
    assert O.mean_f32(a) == z[f"mean.n{n}.m"][0]


def test_philox_and_floyd_restatements():
    seed = O.derive_seed(3, 1, 4, 1)
    u = O.philox_uniforms(seed, 12)
    words = [w for c in (1, 2, 3) for w in O.philox4x64_block(c, O.stream_key(seed))]
    assert [np.float64((w >> 11) * 2.0 ** -53) for w in words] == list(u)
    for n, k in [(20000, 200), (5000, 2500), (10, 10), (44454, 444)]:
        s = O.derive_seed(2, 0, n, k)
        ref = np.sort(O.generator(s).choice(n, size=k, replace=False))
        assert np.array_equal(ref, O.floyd_choice(s, n, k))


def test_payload_bytes_agree():
    from paper_2103_15195_b200.spec import ALGORITHMS, payload_bytes

    for algo in ALGORITHMS:
        for kw in ({}, {"levels": 16, "bucket_size": 50}, {"sparsity": 0.5}):
            spec = CompressorSpec(algo, **kw)
            for n in (1, 7, 63, 512, 1000, 4109, 10 ** 6):
                assert payload_bytes(spec, n) == O.payload_bytes(spec, n)
