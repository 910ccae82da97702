"""world_size-2 multi-process tests of the exchange layer on the gloo backend (CPU):
rank-ordered placement of fixed-size payloads, and the two-phase (counts, then
padded) gather of data-dependent threshold payloads with the re-pack to a common
capacity — the logic the NCCL path runs on the GPUs."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_15195_b200 import exchange


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _sparse_payload(rank, count, cap):
    hdr = torch.zeros(8, dtype=torch.int32)
    hdr[0] = 5  # threshold
    hdr[2] = 1000  # original_len lo
    hdr[4] = count
    hdr[5] = count
    hdr[7] = cap
    body_idx = torch.zeros(exchange._a16(4 * cap) // 4, dtype=torch.int32)
    body_val = torch.zeros(exchange._a16(4 * cap) // 4, dtype=torch.float32)
    body_idx[:count] = torch.arange(count, dtype=torch.int32) * 3 + rank
    body_val[:count] = torch.arange(count, dtype=torch.float32) + 100 * rank
    return torch.cat([hdr.view(torch.uint8), body_idx.view(torch.uint8), body_val.view(torch.uint8)])


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # fixed-size payloads land in rank order
        mine = torch.full((48,), rank + 1, dtype=torch.uint8)
        out, stride = exchange.allgather_fixed(mine)
        assert stride == 48
        for r in range(world):
            assert torch.all(out[r * 48:(r + 1) * 48] == r + 1)
        # variable counts: rank 0 keeps 3, rank 1 keeps 7 (local capacity n = 50)
        count = 3 if rank == 0 else 7
        pay = _sparse_payload(rank, count, 50)
        gathered, stride, counts = exchange.allgather_variable(pay)
        assert counts == [3, 7]
        cap = 7
        assert stride == 32 + 2 * exchange._a16(4 * cap)
        for r in range(world):
            blk = gathered[r * stride:(r + 1) * stride]
            h = blk[:32].view(torch.int32)
            assert int(h[4]) == counts[r] and int(h[7]) == cap
            idx = blk[32:32 + 4 * counts[r]].view(torch.int32)
            voff = 32 + exchange._a16(4 * cap)
            val = blk[voff:voff + 4 * counts[r]].view(torch.float32)
            assert idx.tolist() == [3 * i + r for i in range(counts[r])]
            assert val.tolist() == [float(i + 100 * r) for i in range(counts[r])]
        # the same, through persistent buffers (the GradSync NCCL path: no allocation)
        bufs = {"cnt": torch.zeros(1, dtype=torch.int64), "counts": torch.zeros(world, dtype=torch.int64),
                "mine": torch.zeros(pay.numel(), dtype=torch.uint8),
                "gather": torch.zeros(world * pay.numel(), dtype=torch.uint8)}
        g2, s2, c2 = exchange.allgather_variable(pay, cap_in=50, bufs=bufs)
        assert c2 == counts and s2 == stride and torch.equal(g2, gathered)
        assert g2.data_ptr() == bufs["gather"].data_ptr()
        # dense baseline: in-place sum then / world, equal to aggregate of identity payloads
        x = torch.linspace(-1, 1, 101, dtype=torch.float32) * (rank + 1) / 3
        ref = (torch.linspace(-1, 1, 101, dtype=torch.float32) / 3 + torch.linspace(-1, 1, 101) * 2 / 3) / 2.0
        exchange.allreduce_mean_(x)
        assert torch.equal(x, ref)
        y = torch.full((7,), float(rank))
        work = exchange.allreduce_mean_(y, async_op=True)
        if work is not None:
            work.wait()
            y.div_(2.0)
        assert torch.equal(y, torch.full((7,), 0.5))
        assert exchange.world() == (rank, world)
        q.put((rank, "ok"))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_exchange_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_single_process_exchange_is_identity():
    buf = torch.arange(32, dtype=torch.uint8)
    out, stride = exchange.allgather_fixed(buf)
    assert out is buf and stride == 32
