"""Allgather over peer memory fused with the encode (mc_encode_push / mc_push_wait), checked
on one GPU by simulating N ranks: N gather buffers and N flag arrays live on the device; rank
r encodes its gradient and pushes its payload into slot r of every gather buffer.  Every
gather buffer must equal, byte for byte, the rank-ordered concatenation an NCCL allgather
of independently encoded payloads produces, and decode to the same mean."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("algo", ["efsignsgd", "onebit", "int8", "dgc_lite", "qsgd", "signsgd", "fp16", "threshold"])
@pytest.mark.parametrize("nranks", [2, 4])
def test_encode_push_equals_allgather(algo, nranks):
    from paper_2103_15195_b200 import _native
    from paper_2103_15195_b200 import compressors as C
    from paper_2103_15195_b200.spec import CompressorSpec

    spec = CompressorSpec(algo, sparsity=0.999, threshold=2e-3)
    n = 1_000_003 if algo not in ("efsignsgd", "onebit", "int8") else 1_048_576 + 512 * 7 + 13
    L = _native.layout(spec.to_c(), n)
    stride = (L.bytes + 15) // 16 * 16
    gens = [torch.Generator(device="cuda").manual_seed(100 + r) for r in range(nranks)]
    grads = [torch.randn(n, device="cuda", generator=g) * 1e-3 for g in gens]
    ef = spec.uses_error_feedback
    res_a = [torch.zeros(n, dtype=torch.float64, device="cuda") if ef else None for _ in range(nranks)]
    res_b = [torch.zeros(n, dtype=torch.float64, device="cuda") if ef else None for _ in range(nranks)]
    gather = [torch.zeros(nranks * stride, dtype=torch.uint8, device="cuda") for _ in range(nranks)]
    flags = [torch.zeros(nranks, dtype=torch.int32, device="cuda") for _ in range(nranks)]
    for epoch in (1, 2):  # two exchanges: state carried, flags re-armed by the epoch
        for r in range(nranks):
            own = gather[r][r * stride:(r + 1) * stride]
            dsts = [gather[j].data_ptr() + r * stride for j in range(nranks)]
            fl = [flags[j].data_ptr() + 4 * r for j in range(nranks)]
            C.device_encode_push(spec, grads[r] * epoch, res_a[r], None, 1000 * epoch + r, own, dsts, fl, epoch)
        for j in range(nranks):
            C.push_wait(flags[j], nranks, epoch)
        ref = torch.zeros(nranks * stride, dtype=torch.uint8, device="cuda")
        for r in range(nranks):
            C.device_encode(spec, grads[r] * epoch, res_b[r], None, 1000 * epoch + r, out=ref[r * stride:r * stride + L.bytes])
        torch.cuda.synchronize()
        for j in range(nranks):
            if algo == "threshold":  # the push moves header + the first n_idx entries only
                for r in range(nranks):
                    a, b = gather[j][r * stride:(r + 1) * stride], ref[r * stride:(r + 1) * stride]
                    cnt = int(b[16:20].view(torch.int32).item())
                    assert 0 < cnt < n and torch.equal(a[:32], b[:32])
                    for off in (L.off_idx, L.off_val):
                        assert torch.equal(a[off:off + 4 * cnt], b[off:off + 4 * cnt]), (epoch, j, r)
            else:
                assert torch.equal(gather[j], ref), (algo, nranks, epoch, j)
        if ef:
            for r in range(nranks):
                assert torch.equal(res_a[r].view(torch.int64), res_b[r].view(torch.int64))
        outs = []
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        for j in range(nranks):
            o = torch.empty(n, device="cuda")
            C.device_decode_mean(spec, gather[j], stride, nranks, n, o, err)
            outs.append(o)
        torch.cuda.synchronize()
        assert int(err.item()) == 0
        for o in outs[1:]:
            assert torch.equal(o.view(torch.int32), outs[0].view(torch.int32))


@pytest.mark.parametrize("case", ["ragged", "resnet50"])
def test_merge_stage_pack_unpack(case):
    """K1 / K11 (trainer.py:344-348 as a copy): mc_pack == torch.cat, mc_unpack its inverse,
    for ragged sizes (zero-length tensors, 8192-element chunk edges, every 16-byte phase of
    source vs fused offset) and the 161 ResNet-50 tensors (> 128: one launch since PACK_MAX=512)."""
    from paper_2103_15195_b200 import gradsets, merge

    if case == "ragged":  # empty tensors, 8192-element chunk edges
        sizes = [1, 3, 4, 5, 8191, 8192, 8193, 0, 17, 100_000]
    else:
        sizes = list(gradsets.sizes("resnet50_161"))
    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(5)
    # sub-views at odd element offsets make the sources' 16-byte phase differ from the fused one
    backing = [torch.randn(n + 3, generator=g).to(dev) for n in sizes]
    srcs = [b[1 + (i % 3): 1 + (i % 3) + n] for i, (b, n) in enumerate(zip(backing, sizes))]
    fused = merge.pack(srcs)
    ref = torch.cat([s.reshape(-1) for s in srcs])
    assert torch.equal(fused, ref)
    outs = [torch.full((n,), float("nan"), device=dev) for n in sizes]
    merge.unpack(fused * 2, outs)
    torch.cuda.synchronize()
    for o, s in zip(outs, srcs):
        assert torch.equal(o, s * 2)


class _Ptr:
    """A raw device address with the tensor interface the decode wrappers read."""

    def __init__(self, addr):
        self.addr = addr

    def data_ptr(self):
        return self.addr


@pytest.mark.parametrize("algo", ["efsignsgd", "onebit", "int8"])
@pytest.mark.parametrize("nranks", [1, 2, 4])
def test_multicast_push_equals_allgather(algo, nranks):
    """The NVLS push (mc_encode_push_mc): one multicast object on this GPU holds the gather
    buffer and the flag words; N simulated ranks each store their payload ONCE through
    their slot's multicast address (multimem.st) and release their flag the same way.  The
    device's unicast view must equal, byte for byte, the rank-ordered concatenation of
    independently encoded payloads, the flags must carry the epoch, and the decode must
    equal the plain decode_mean."""
    from cuda.bindings import runtime as cudart

    from paper_2103_15195_b200 import _native
    from paper_2103_15195_b200 import compressors as C
    from paper_2103_15195_b200.spec import CompressorSpec

    spec = CompressorSpec(algo)
    n = 1_048_576 + 512 * 7 + 13
    L = _native.layout(spec.to_c(), n)
    stride = (L.bytes + 15) // 16 * 16
    foff = nranks * stride
    try:
        buf = C.McastBuffer([0], foff + 4 * nranks)
    except _native.NativeError as exc:  # e.g. cuMulticastCreate rejected (no NVLS fabric on this box)
        pytest.skip(f"multicast objects unavailable here: {exc}")
    cudart.cudaMemset(buf.unicast[0], 0, buf.nbytes)
    gens = [torch.Generator(device="cuda").manual_seed(500 + r) for r in range(nranks)]
    grads = [torch.randn(n, device="cuda", generator=g) * 1e-3 for g in gens]
    ef = spec.uses_error_feedback
    res_a = [torch.zeros(n, dtype=torch.float64, device="cuda") if ef else None for _ in range(nranks)]
    res_b = [torch.zeros(n, dtype=torch.float64, device="cuda") if ef else None for _ in range(nranks)]
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    try:
        for epoch in (1, 2):
            for r in range(nranks):
                C.device_encode_push_mc(spec, grads[r] * epoch, res_a[r], None, 1, buf.unicast[0] + r * stride,
                                        buf.multicast + r * stride, buf.multicast + foff + 4 * r, epoch, err)
            flags = torch.empty(nranks, dtype=torch.int32, device="cuda")
            C.push_wait(_FlagView(buf.unicast[0] + foff), nranks, epoch, err, timeout_s=20.0)
            got = torch.empty(foff, dtype=torch.uint8, device="cuda")
            torch.cuda.synchronize()
            cudart.cudaMemcpy(got.data_ptr(), buf.unicast[0], foff, cudart.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
            cudart.cudaMemcpy(flags.data_ptr(), buf.unicast[0] + foff, 4 * nranks,
                              cudart.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
            ref = torch.zeros(foff, dtype=torch.uint8, device="cuda")
            for r in range(nranks):
                C.device_encode(spec, grads[r] * epoch, res_b[r], None, 1, out=ref[r * stride:r * stride + L.bytes])
            torch.cuda.synchronize()
            assert int(err.item()) == 0
            assert bool((flags == epoch).all())
            for r in range(nranks):  # payload bytes of every slot (the slot tails are padding)
                assert torch.equal(got[r * stride:r * stride + L.bytes], ref[r * stride:r * stride + L.bytes]), (algo, r)
            if ef:
                for r in range(nranks):
                    assert torch.equal(res_a[r].view(torch.int64), res_b[r].view(torch.int64))
            o1, o2 = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
            C.device_decode_mean(spec, _Ptr(buf.unicast[0]), stride, nranks, n, o1, err)
            C.device_decode_mean(spec, ref, stride, nranks, n, o2, err)
            torch.cuda.synchronize()
            assert torch.equal(o1.view(torch.int32), o2.view(torch.int32))
    finally:
        buf.close()


class _FlagView(_Ptr):
    device = torch.device("cuda", 0)
