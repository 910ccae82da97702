"""GPU parity of the sync engine (GradSync) against the oracle's Trainer.step group
loop (trainer.py:376-389): per group encode with per-(boundaries, worker, group)
state and derive_seed(root, rank, iteration, group) keys, then aggregate — the
averaged gradients and the fp64 residuals bit for bit over several iterations."""

import numpy as np
import pytest

import mergecomp_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SPECS = [
    dict(algorithm="efsignsgd"),
    dict(algorithm="onebit"),
    dict(algorithm="int8"),
    dict(algorithm="qsgd"),
    dict(algorithm="terngrad"),
    dict(algorithm="dgc_lite", sparsity=0.99),
    dict(algorithm="topk", sparsity=0.9),
    dict(algorithm="randk", sparsity=0.99),
    dict(algorithm="randk", sparsity=0.99, error_feedback=True, momentum=0.9, unbiased_scaling=True),
    dict(algorithm="randk", sparsity=0.95, error_feedback=True),
    dict(algorithm="randk", sparsity=0.99, momentum=0.5),
    dict(algorithm="threshold", threshold=2e-3),
    dict(algorithm="signsgd"),
    dict(algorithm="signum"),
    dict(algorithm="fp16"),
    dict(algorithm="identity"),
    dict(algorithm="efsignsgd", bucket_size=256, error_feedback=False),
    dict(algorithm="efsignsgd", bucket_size=50),
]


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


@pytest.mark.parametrize("kw", SPECS, ids=lambda k: "-".join(f"{v}" for v in k.values()))
@pytest.mark.parametrize("fused", [True, False])
def test_gradsync_matches_oracle_trainer_loop(kw, fused):
    from paper_2103_15195_b200 import gradsets
    from paper_2103_15195_b200.profiles import Partition
    from paper_2103_15195_b200.spec import CompressorSpec
    from paper_2103_15195_b200.sync import GradSync

    spec = CompressorSpec(**kw)
    prof = gradsets.profile("tiny40")
    part = Partition(prof.n_tensors, (5, 23))
    sync = GradSync(spec, prof, partition=part, root_seed=11)
    sync.fuse_local = fused
    ranges = part.element_ranges(prof)
    states = {}
    for it in range(3):
        g = gradsets.synthetic_gradients("tiny40", it, 0)
        sync.flat.copy_(torch.from_numpy(g))
        sync.step()
        torch.cuda.synchronize()
        sync.check()
        for gi, (a, b) in enumerate(ranges):
            mean, _, new = O.sync_group(spec, [g[a:b]], [states.get(gi)], [O.derive_seed(11, 0, it, gi)])
            states[gi] = new[0]
            got = sync.flat[a:b].cpu().numpy()
            assert np.array_equal(_bits(got), _bits(mean)), f"{spec.algorithm} it{it} group{gi} mean"
            plan = sync._plan(part)[gi]
            if plan.residual is not None:
                assert np.array_equal(_bits(plan.residual.cpu().numpy()), _bits(new[0].residual)), "residual"


def test_fused_path_on_resnet50_group(rng=None):
    """The TMA-pipelined fused encode+decode on a full ResNet-50 gradient set (25.6M)
    equals encode followed by decode_mean, bit for bit (payload, residual, output)."""
    from paper_2103_15195_b200 import compressors as C
    from paper_2103_15195_b200 import gradsets
    from paper_2103_15195_b200.spec import CompressorSpec

    g = torch.from_numpy(gradsets.synthetic_gradients("resnet50_161", 0, 0)).cuda()
    for algo in ("efsignsgd", "onebit", "int8", "qsgd", "terngrad"):
        spec = CompressorSpec(algo, error_feedback=True)
        r1 = torch.zeros(g.numel(), dtype=torch.float64, device="cuda")
        r1.normal_(0, 1e-4)
        r2 = r1.clone()
        out = g.clone()
        p1 = C.device_encode_decode(spec, out, r1, None, 5, out)  # in place
        p2 = C.device_encode(spec, g, r2, None, 5)
        ref = torch.empty_like(g)
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        C.device_decode_mean(spec, p2.buf, p2.buf.numel(), 1, g.numel(), ref, err)
        torch.cuda.synchronize()
        assert int(err.item()) == 0
        s1, s2 = p1.canonical_sections(), p2.canonical_sections()  # padding bytes are unspecified
        for a, b in zip(s1, s2):
            assert (a is None and b is None) or torch.equal(a, b), f"{algo} payload"
        assert torch.equal(r1.view(torch.int64), r2.view(torch.int64)), f"{algo} residual"
        assert torch.equal(out.view(torch.int32), ref.view(torch.int32)), f"{algo} out"


def test_large_group_against_oracle():
    """One 2M-element group (> one TMA tile per SM) vs the oracle, EF over 2 iterations."""
    from paper_2103_15195_b200 import compressors as C
    from paper_2103_15195_b200.spec import CompressorSpec

    rng = np.random.default_rng(5)
    for algo in ("efsignsgd", "onebit", "qsgd"):
        spec = CompressorSpec(algo, error_feedback=True)
        st_d, st_o = None, None
        for it in range(2):
            x = (rng.standard_normal(2_000_003) * 1e-3).astype(np.float32)
            seed = C.derive_seed(1, 0, it, 0)
            p, st_d = C.encode(spec, torch.from_numpy(x).cuda(), st_d, seed=seed)
            q, st_o = O.encode(spec, x, st_o, seed=seed)
            h = p.to_host()
            assert np.array_equal(_bits(h.values), _bits(q.values)), algo
            assert np.array_equal(h.bits, q.bits), algo
            assert np.array_equal(_bits(st_d.residual.cpu().numpy()), _bits(st_o.residual)), algo


@pytest.mark.parametrize("algo", ["efsignsgd", "onebit", "int8", "fp16", "identity", "qsgd", "dgc_lite", "topk",
                                  "terngrad", "signsgd", "signum", "randk", "threshold"])
def test_sync_host_pipelined_equals_device_step(algo):
    """GradSync.sync_host (chunked H2D / fused encode / D2H pipeline) == device step()."""
    from paper_2103_15195_b200 import gradsets
    from paper_2103_15195_b200.profiles import Partition
    from paper_2103_15195_b200.spec import CompressorSpec
    from paper_2103_15195_b200.sync import GradSync

    spec = CompressorSpec(algo, sparsity=0.99)
    prof = gradsets.profile("resnet50_161")
    part = Partition(prof.n_tensors, (100,))
    a = GradSync(spec, prof, partition=part, root_seed=1)
    b = GradSync(spec, prof, partition=part, root_seed=1)
    for it in range(2):
        g = torch.from_numpy(gradsets.synthetic_gradients("resnet50_161", it, 0)).pin_memory()
        out = a.sync_host(g, chunk_elems=1 << 20)
        b.flat.copy_(g)
        b.step()
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int32), b.flat.cpu().view(torch.int32)), (algo, it)
        for ga, gb in zip(a._plan(part), b._plan(part)):
            if ga.residual is not None:
                assert torch.equal(ga.residual.view(torch.int64), gb.residual.view(torch.int64))


@pytest.mark.parametrize("algo", ["efsignsgd", "dgc_lite", "qsgd"])
def test_backward_overlap_hooks_equal_post_backward_step(algo):
    """WFBP: groups synced from post-accumulate-grad hooks during backward produce the
    same averaged gradients (bitwise) as one step() after backward."""
    torchvision = pytest.importorskip("torchvision")
    from paper_2103_15195_b200.profiles import ModelProfile, Partition
    from paper_2103_15195_b200.spec import CompressorSpec
    from paper_2103_15195_b200.sync import GradSync

    torch.manual_seed(0)
    torch.backends.cudnn.deterministic = True  # both backward passes must produce identical bits
    torch.backends.cudnn.benchmark = False
    spec = CompressorSpec(algo, sparsity=0.99)

    def build():
        torch.manual_seed(0)
        m = torchvision.models.resnet18(weights=None).cuda()
        params = [p for p in m.parameters() if p.requires_grad][::-1]  # backprop order
        prof = ModelProfile.from_sizes("resnet18", [p.numel() for p in params])
        return m, params, prof

    x = torch.randn(8, 3, 64, 64, device="cuda")
    m1, p1, prof = build()
    m2, p2, _ = build()
    part = Partition(prof.n_tensors, (20, 45))
    s1 = GradSync(spec, prof, partition=part, root_seed=4)
    s2 = GradSync(spec, prof, partition=part, root_seed=4)
    s1.attach(p1)
    for it in range(2):
        m1.zero_grad(set_to_none=False)
        s1.begin_backward()
        m1(x).square().mean().backward()
        s1.finish_backward()
        m2.zero_grad(set_to_none=True)
        m2(x).square().mean().backward()
        s2.flat.copy_(torch.cat([p.grad.reshape(-1) for p in p2]))
        s2.step()
        torch.cuda.synchronize()
        assert torch.equal(s1.flat.view(torch.int32), s2.flat.view(torch.int32)), (algo, it)
        assert all(g1.data_ptr() == s1.flat[a:a + 1].data_ptr() for g1, a in zip([p.grad for p in p1], prof.offsets()[:-1]))
    s1.detach()


@pytest.mark.parametrize("wait", [True, False], ids=["joined", "overlapped"])
@pytest.mark.parametrize("algo", ["efsignsgd", "dgc_lite", "qsgd"])
def test_sync_host_back_to_back_calls(algo, wait):
    """Consecutive native host syncs enqueued without a host synchronisation in between
    (each call's H2D chases the previous call's read-out chunk by chunk; overlapped: no call
    joins the current stream until sync_host_wait) give the same outputs as synchronised
    device steps."""
    from paper_2103_15195_b200 import gradsets
    from paper_2103_15195_b200.spec import CompressorSpec
    from paper_2103_15195_b200.sync import GradSync

    spec = CompressorSpec(algo, sparsity=0.999)
    prof = gradsets.profile("resnet50_161")
    a = GradSync(spec, prof, root_seed=3)
    b = GradSync(spec, prof, root_seed=3)
    ins = [torch.from_numpy(gradsets.synthetic_gradients("resnet50_161", it, 0)).pin_memory() for it in range(3)]
    outs = [torch.empty_like(x).pin_memory() for x in ins]
    for x, o in zip(ins, outs):
        a.sync_host(x, o, chunk_elems=1 << 19, wait=wait)
    a.sync_host_wait()
    torch.cuda.synchronize()
    for x, o in zip(ins, outs):
        b.flat.copy_(x)
        b.step()
        torch.cuda.synchronize()
        assert torch.equal(o.view(torch.int32), b.flat.cpu().view(torch.int32))


ALL_CODECS = ["identity", "fp16", "topk", "dgc_lite", "randk", "threshold", "qsgd", "signsgd", "signum", "efsignsgd",
              "onebit", "terngrad", "int8"]


@pytest.mark.parametrize("algo", ALL_CODECS)
def test_graph_replay_equals_eager_steps(algo):
    """A CUDA Graph of a pinned many-group partition replays to the same averaged
    gradients and codec state (bitwise) as eager steps — all 13 codecs: the stochastic
    ones draw their per-(iteration, group) Philox keys on the device inside the graph."""
    from paper_2103_15195_b200 import gradsets
    from paper_2103_15195_b200.scheduler import naive_partition
    from paper_2103_15195_b200.spec import CompressorSpec
    from paper_2103_15195_b200.sync import GradSync

    spec = CompressorSpec(algo, sparsity=0.99 if algo == "randk" else 0.999)
    prof = gradsets.profile("resnet50_161")
    part = naive_partition(prof.n_tensors, 12)
    a = GradSync(spec, prof, partition=part, root_seed=5)
    b = GradSync(spec, prof, partition=part, root_seed=5)
    a.step()  # one eager step first: the graph continues the iteration count from the host
    b.step()
    a.capture_graph()
    other = naive_partition(prof.n_tensors, 3)
    for it in range(4):
        g = torch.from_numpy(gradsets.synthetic_gradients("resnet50_161", it, 0)).cuda()
        a.flat.copy_(g)
        b.flat.copy_(g)
        if it == 2:  # an eager step of another partition in between: the keys follow the iteration
            a.step(other)
            b.step(other)
            a.flat.copy_(g)
            b.flat.copy_(g)
        a.step()
        b.step()
        torch.cuda.synchronize()
        assert torch.equal(a.flat.view(torch.int32), b.flat.view(torch.int32)), (algo, it)
        for ga, gb in zip(a._plan(part), b._plan(part)):
            if ga.residual is not None:
                assert torch.equal(ga.residual.view(torch.int64), gb.residual.view(torch.int64))
            if ga.momentum is not None:
                assert torch.equal(ga.momentum.view(torch.int32), gb.momentum.view(torch.int32))


def test_drop_state_releases_captured_graph_and_caps_cached_plans():
    """a CUDA Graph captured over a partition's buffers must die with them, and a
    measured search must not keep every candidate's fp64 residual alive."""
    from paper_2103_15195_b200 import gradsets
    from paper_2103_15195_b200.profiles import Partition
    from paper_2103_15195_b200.spec import CompressorSpec
    from paper_2103_15195_b200.sync import GradSync

    prof = gradsets.profile("tiny40")
    sync = GradSync(CompressorSpec("efsignsgd"), prof, partition=Partition(prof.n_tensors, (7,)))
    sync.capture_graph()
    assert sync._graph is not None
    sync.drop_state(Partition(prof.n_tensors, (7,)))
    assert sync._graph is None and not sync._plans
    sync.step()  # eager again, fresh zero state
    for cut in range(1, 20):  # a search visiting 19 candidates
        sync.timed_iteration(Partition(prof.n_tensors, (cut,)))
    assert len(sync._plans) <= GradSync.MAX_CACHED_PLANS + 1
    assert sync.partition.boundaries in sync._plans


def test_nonfinite_gradient_leaves_no_nan_state():
    """encode() never mutates the caller's device state (the reference raises
    before touching it), and the engine resets the poisoned EF state when check() raises."""
    from paper_2103_15195_b200 import compressors as C
    from paper_2103_15195_b200 import gradsets
    from paper_2103_15195_b200.spec import CompressorSpec
    from paper_2103_15195_b200.sync import GradSync

    spec = CompressorSpec("efsignsgd")
    x = torch.randn(10_000, device="cuda")
    _, st = C.encode(spec, x, None)
    before = st.residual.clone()
    bad = x.clone()
    bad[17] = float("nan")
    with pytest.raises(ValueError, match="non-finite"):
        C.encode(spec, bad, st)
    assert torch.equal(st.residual.view(torch.int64), before.view(torch.int64))
    _, st2 = C.encode(spec, x, st)
    assert st2.residual is not st.residual  # a new state object, as in the reference

    prof = gradsets.profile("tiny40")
    sync = GradSync(spec, prof)
    sync.flat.copy_(torch.from_numpy(gradsets.synthetic_gradients("tiny40", 0, 0)))
    sync.flat[5] = float("inf")
    sync.step()
    with pytest.raises(ValueError, match="non-finite"):
        sync.check()
    res = sync._plan(sync.partition)[0].residual
    assert bool(torch.isfinite(res).all()) and not bool(res.any())
    sync.flat.copy_(torch.from_numpy(gradsets.synthetic_gradients("tiny40", 1, 0)))
    sync.step()
    sync.check()
    assert bool(torch.isfinite(sync.flat).all())
