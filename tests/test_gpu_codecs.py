"""GPU parity: every codec through the C ABI on the B200 against the golden vectors
recorded from the reference (tests/golden) — payload sections, fp64 residuals,
fp32 momentum and the rank-ordered mean, bit for bit.  Multi-worker cases stack
the workers' device payloads into one gather buffer and run mc_decode_mean over
it, exactly as the NCCL allgather output is consumed on every rank."""

import numpy as np
import pytest

import golden_cases as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TIE_CASES = {"topk_dyadic_ef"}


def _eq_bits(dev, ref, what):
    a = np.ascontiguousarray(dev)
    b = np.ascontiguousarray(ref)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    if a.dtype.kind == "f":
        # NaN payload bits are not specified by IEEE 754 (x86 yields the negative default
        # NaN, CUDA the positive canonical one): NaN positions must agree, bits elsewhere.
        na, nb = np.isnan(a), np.isnan(b)
        assert np.array_equal(na, nb), f"{what}: NaN positions differ"
        a, b = np.where(na, 0, a).astype(a.dtype), np.where(nb, 0, b).astype(b.dtype)
    if not np.array_equal(a.view(np.uint8), b.view(np.uint8)):
        diff = np.flatnonzero((a.view(np.uint8).reshape(a.size, -1) != b.view(np.uint8).reshape(b.size, -1)).any(axis=1))
        raise AssertionError(f"{what}: {len(diff)} of {a.size} differ, first {diff[:8]}: {a.ravel()[diff[:4]]} vs {b.ravel()[diff[:4]]}")


@pytest.fixture(scope="module")
def C():
    from paper_2103_15195_b200 import compressors

    return compressors


@pytest.mark.parametrize("cid", G.case_ids())
def test_device_path_matches_reference(cid, C):
    from paper_2103_15195_b200.spec import CompressorSpec

    c = G.get_case(cid)
    spec = CompressorSpec(**c["spec"])
    xs = G.inputs(c)
    dev = torch.device("cuda")
    W = c["workers"]
    states = [None] * W
    for t in range(c["iters"]):
        payloads = []
        for w in range(W):
            x = torch.from_numpy(xs[t][w]).to(dev)
            p, s = C.encode(spec, x, states[w], seed=G.seed(cid, t, w))
            states[w] = s
            payloads.append(p)
            h = p.to_host()
            if cid in TIE_CASES:
                assert len(h.indices) == len(G.field(cid, t, w, "idx"))
                continue
            for name, got in (("idx", h.indices), ("val", h.values), ("bits", h.bits)):
                ref = G.field(cid, t, w, name)
                if ref is None:
                    assert got is None or len(got) == 0, (cid, name)
                else:
                    _eq_bits(got, ref, f"{cid} t{t} w{w} {name}")
            assert h.flags == int(G.field(cid, t, w, "flags")[0])
            res = G.field(cid, t, w, "res")
            if res is not None:
                _eq_bits(s.residual.cpu().numpy(), res, f"{cid} t{t} w{w} residual")
            mom = G.field(cid, t, w, "mom")
            if mom is not None:
                _eq_bits(s.momentum.cpu().numpy(), mom, f"{cid} t{t} w{w} momentum")
            ser = G.field(cid, t, w, "ser")
            if ser is not None:
                assert C.serialize(p) == ser.tobytes(), f"{cid} serialize"
        mean = C.aggregate(spec, payloads)
        if cid not in TIE_CASES:
            _eq_bits(mean.cpu().numpy(), G.mean(cid, t), f"{cid} t{t} mean")


@pytest.mark.parametrize("cid", ["efsignsgd_n1000", "qsgd_zeros_w2", "topk_ef_w3", "threshold_tau05", "randk_small_n",
                                 "onebit_b50", "int8_b7", "fp16_range", "signum_mom"])
def test_host_arrays_drop_in(cid, C):
    """numpy in -> numpy out through the same GPU kernels (the reference's calling convention)."""
    from paper_2103_15195_b200.spec import CompressorSpec

    c = G.get_case(cid)
    spec = CompressorSpec(**c["spec"])
    xs = G.inputs(c)
    states = [None] * c["workers"]
    for t in range(c["iters"]):
        payloads = []
        for w in range(c["workers"]):
            p, states[w] = C.encode(spec, xs[t][w], states[w], seed=G.seed(cid, t, w))
            assert isinstance(p.values, np.ndarray)
            _eq_bits(p.values, G.field(cid, t, w, "val"), f"{cid} val")
            payloads.append(p)
        mean = C.aggregate(spec, payloads)
        assert isinstance(mean, np.ndarray)
        _eq_bits(mean, G.mean(cid, t), f"{cid} mean")


def test_non_finite_rejected(C):
    from paper_2103_15195_b200.spec import CompressorSpec

    with pytest.raises(ValueError, match="finite"):
        C.encode(CompressorSpec("identity"), np.float32([1.0, np.nan]))
    with pytest.raises(ValueError, match="finite"):
        C.encode(CompressorSpec("efsignsgd"), torch.tensor([1.0, float("inf")] * 300, device="cuda"))


def test_corrupt_indices_rejected(C):
    from paper_2103_15195_b200.spec import CompressorSpec

    spec = CompressorSpec("topk", error_feedback=False)
    bad = C.CompressedPayload("topk", 4, np.array([7], np.uint32), np.float32([1.0]), None)
    with pytest.raises(ValueError, match="corrupt"):
        C.decode(spec, bad)
    bad2 = C.CompressedPayload("topk", 8, np.array([3, 1], np.uint32), np.float32([1.0, 2.0]), None)
    with pytest.raises(ValueError, match="corrupt"):
        C.decode(spec, bad2)


def test_derive_seed_native_matches_table(C):
    for root, w, t, g, lo, hi in G.store()["derive_seed.table"].tolist():
        assert C.derive_seed(root, w, t, g) == (lo | (hi << 64))


@pytest.mark.parametrize("sparsity,sigma", [(0.99, None), (0.999, None), (0.99, "2"), (0.98, "3")])
def test_randk_resnet50_size_matches_oracle(sparsity, sigma, C, monkeypatch):
    """randk over a whole ResNet-50-sized group (25.56M elements, ~250 windows at 1%): the
    5-launch path (tables, link, draw emit, Floyd, persistent emit) and, with a narrow band,
    its hybrid serial fallback — indices and values bit-exact against numpy's choice."""
    import torch

    import mergecomp_oracle as O
    from paper_2103_15195_b200.spec import CompressorSpec

    if sigma is not None:
        monkeypatch.setenv("MC_RANDK_BAND_SIGMA", sigma)
    n = 25_557_032
    spec = CompressorSpec("randk", sparsity=sparsity)
    g = (np.random.default_rng(17).standard_normal(n) * 1e-3).astype(np.float32)
    seed = O.derive_seed(5, 0, 7, 0)
    p_dev, _ = C.encode(spec, torch.from_numpy(g).cuda(), None, seed=seed)
    p_ref, _ = O.encode(spec, g, None, seed=seed)
    d = p_dev.to_host()
    assert np.array_equal(np.asarray(d.indices), np.asarray(p_ref.indices))
    assert np.array_equal(np.asarray(d.values).view(np.uint32), np.asarray(p_ref.values).view(np.uint32))


@pytest.mark.parametrize("sigma", ["0", "1.5"])
def test_randk_serial_fallback_matches_oracle(sigma, C, monkeypatch):
    """A speculated-offset band too narrow for the walk's drift (MC_RANDK_BAND_SIGMA, a test
    knob) makes the chain leave a window's range: the link kernel's last CTA then walks the rest
    of the stream serially.  Results must not change (bit-exact vs the oracle)."""
    import torch

    import mergecomp_oracle as O
    from paper_2103_15195_b200.spec import CompressorSpec

    monkeypatch.setenv("MC_RANDK_BAND_SIGMA", sigma)
    n = 4_000_037
    spec = CompressorSpec("randk", sparsity=0.99)
    g = (np.random.default_rng(5).standard_normal(n) * 1e-3).astype(np.float32)
    seed = O.derive_seed(11, 1, 2, 0)
    p_dev, _ = C.encode(spec, torch.from_numpy(g).cuda(), None, seed=seed)
    p_ref, _ = O.encode(spec, g, None, seed=seed)
    d = p_dev.to_host()
    assert np.array_equal(np.asarray(d.indices), np.asarray(p_ref.indices))
    assert np.array_equal(np.asarray(d.values).view(np.uint32), np.asarray(p_ref.values).view(np.uint32))


@pytest.mark.parametrize("n,sparsity", [(2_000_003, 0.99), (3_000_000, 0.995), (1_500_000, 0.9)])
def test_randk_multi_window_walk_matches_oracle(n, sparsity, C):
    """randk at sizes where the draw walk spans many 1024-position windows (speculative
    tables + chain + emit on many SMs; 0.9 takes numpy's tail-shuffle branch): indices and
    values bit-exact against the oracle's Generator.choice restatement."""
    import torch

    import mergecomp_oracle as O
    from paper_2103_15195_b200.spec import CompressorSpec

    spec = CompressorSpec("randk", sparsity=sparsity)
    rng = np.random.default_rng(n)
    g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    seed = O.derive_seed(7, 0, 3, 1)
    p_dev, _ = C.encode(spec, torch.from_numpy(g).cuda(), None, seed=seed)
    p_ref, _ = O.encode(spec, g, None, seed=seed)
    d = p_dev.to_host()
    assert np.array_equal(np.asarray(d.indices), np.asarray(p_ref.indices))
    assert np.array_equal(np.asarray(d.values).view(np.uint32), np.asarray(p_ref.values).view(np.uint32))


@pytest.mark.parametrize("n", [25_557_032, 120_000_001])
def test_signsgd_large_group_scale_matches_numpy(n, C):
    """signsgd's scaler over a whole large group (numpy's float32 pairwise mean): node
    trees of ~800 (depth-3 leaves) and ~920 elements (depth-4) — the scale bit-exact, and
    the sign bits equal np.packbits(x >= 0)."""
    import torch

    from paper_2103_15195_b200.spec import CompressorSpec

    rng = np.random.default_rng(n)
    x = rng.standard_normal(n, dtype=np.float32) * np.float32(1e-3)
    p, _ = C.encode(CompressorSpec("signsgd"), torch.from_numpy(x).cuda(), None, seed=0)
    h = p.to_host()
    want = np.float32(np.abs(x).mean())
    assert np.asarray(h.values).view(np.uint32)[0] == np.asarray([want]).view(np.uint32)[0]
    assert np.array_equal(np.asarray(h.bits), np.packbits(x >= 0))


@pytest.mark.parametrize("algo,ef", [("qsgd", False), ("qsgd", True), ("terngrad", False), ("int8", False),
                                     ("int8", True)])
def test_quantizer_scale_range_matches_oracle(algo, ef, C):
    """The quantizers divide by the bucket scale with the reciprocal hoisted per bucket and
    the IEEE fast path inline; elements or scales outside [2^-40, 2^40] take the full
    division.  Magnitudes from 2^-70 to 2^60, whole buckets of tiny / huge values and
    exact zeros: codes, scales and residuals bit-exact against the oracle."""
    import torch

    import mergecomp_oracle as O
    from paper_2103_15195_b200.spec import CompressorSpec

    rng = np.random.default_rng(2103)
    n = 512 * 400 + 77
    e = rng.uniform(-70, 20, n)
    g = (np.sign(rng.standard_normal(n)) * rng.uniform(1, 2, n) * np.exp2(e)).astype(np.float32)
    g[512 * 3:512 * 4] = (rng.standard_normal(512) * 2.0 ** -50).astype(np.float32)  # scale < 2^-40
    g[512 * 7:512 * 8] = (rng.standard_normal(512) * 2.0 ** 55).astype(np.float32)   # scale > 2^40
    g[512 * 9:512 * 10] = 0.0
    g[rng.integers(0, n, 500)] = 0.0
    g[rng.integers(0, n, 200)] = -0.0
    spec = CompressorSpec(algo, error_feedback=ef, bucket_size=512)
    st_d, st_r = None, None
    for t in range(2):
        seed = O.derive_seed(11, 0, t, 0)
        p_dev, st_d = C.encode(spec, torch.from_numpy(g).cuda(), st_d, seed=seed)
        p_ref, st_r = O.encode(spec, g, st_r, seed=seed)
        d = p_dev.to_host()
        for name in ("values", "bits"):
            a, b = getattr(d, name), getattr(p_ref, name)
            if b is None:
                assert a is None or len(a) == 0
            else:
                _eq_bits(np.asarray(a), np.asarray(b), f"{algo} t{t} {name}")
        if ef:
            _eq_bits(st_d.residual.cpu().numpy(), np.asarray(st_r.residual), f"{algo} t{t} residual")
        _eq_bits(C.aggregate(spec, [p_dev]).cpu().numpy(), np.asarray(O.aggregate(spec, [p_ref])), f"{algo} t{t} mean")


@pytest.mark.parametrize("algo", ["identity", "fp16", "topk", "randk", "dgc_lite", "threshold", "qsgd", "signsgd",
                                  "efsignsgd", "onebit", "signum", "terngrad", "int8"])
def test_serialize_deserialize_roundtrip_on_device(algo, C):
    """Acceptance #8(d) (test_acceptance.py:283-291) through the device ABI: the canonical
    bytes from mc_serialize, parsed back by mc_deserialize (and by the host deserialize),
    decode to the same gradient and re-serialize to the same bytes."""
    from paper_2103_15195_b200.spec import CompressorSpec

    spec = CompressorSpec(algo, error_feedback=False)
    rng = np.random.default_rng(8)
    for n in (1, 63, 513, 2048, 100_003):
        x = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).cuda()
        p, _ = C.encode(spec, x, seed=3)
        raw = C.serialize(p)
        assert len(raw) == p.byte_size
        back_d = C.device_deserialize(spec, raw)
        back_h = C.deserialize(raw)
        assert back_d.on_device and not back_h.on_device
        ref = C.decode(spec, p).cpu().numpy()
        assert np.array_equal(C.decode(spec, back_d).cpu().numpy().view(np.uint32), ref.view(np.uint32)), (algo, n)
        assert np.array_equal(np.asarray(C.decode(spec, back_h)).view(np.uint32), ref.view(np.uint32)), (algo, n)
        assert C.serialize(back_d) == raw, (algo, n)
        assert C.serialize(back_h) == raw, (algo, n)
    # malformed input: the reference's errors (compressors.py:623-645)
    with pytest.raises(ValueError, match="shorter than header"):
        C.device_deserialize(spec, raw[:10])
    with pytest.raises(ValueError, match="does not match header"):
        C.device_deserialize(spec, raw + b"\0")
    with pytest.raises(ValueError, match="unknown algorithm id"):
        C.device_deserialize(spec, bytes([99]) + raw[1:])


@pytest.mark.parametrize("algo,bucket", [("efsignsgd", 512), ("efsignsgd", 384), ("onebit", 512), ("onebit", 128),
                                         ("signsgd", 512), ("signum", 512), ("int8", 512), ("int8", 136),
                                         ("fp16", 512), ("identity", 512), ("terngrad", 512)])
@pytest.mark.parametrize("nranks", [2, 3, 5, 8, 9])
def test_sign_decode_mean_many_ranks_matches_oracle(algo, bucket, nranks, C):
    """decode_mean over 2..9 stacked payloads against the oracle's rank-ordered aggregate,
    bit for bit: sign codecs (3..8 ranks take the per-bucket table kernel, 2 and 9 the
    per-element loop) and the byte codecs (chunk-prefetching kernel, ragged tail group).
    Ranks differ in magnitude by up to 10^4 so the f32 addition order is visible; the group
    length leaves a partial word and a partial bucket; some buckets are all zero."""
    import torch

    import mergecomp_oracle as O
    from paper_2103_15195_b200.spec import CompressorSpec

    spec = CompressorSpec(algo, bucket_size=bucket)
    n = 200_003
    rng = np.random.default_rng(nranks * 1000 + bucket)
    pays_d, pays_o = [], []
    for r in range(nranks):
        g = (rng.standard_normal(n) * (1e-3 * 10.0 ** ((r % 5) - 2))).astype(np.float32)
        g[4096:4096 + 3 * bucket] = 0.0  # all-zero buckets (sign bit 1, scale 0)
        g[7] = -0.0
        p, _ = C.encode(spec, torch.from_numpy(g).cuda(), None, seed=r + 1)
        q, _ = O.encode(spec, g, None, seed=r + 1)
        pays_d.append(p)
        pays_o.append(q)
    mean_d = C.aggregate(spec, pays_d).cpu().numpy()
    mean_o = O.aggregate(spec, pays_o)
    _eq_bits(mean_d, mean_o, f"{algo} B={bucket} N={nranks} mean")
