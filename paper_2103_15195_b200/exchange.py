"""Payload exchange between data-parallel ranks (the reference's in-memory list,
trainer.py:377-389, becomes an allgather of device payload buffers).

* fixed-size codecs: one ``all_gather_into_tensor`` of the aligned payload
  buffer; rank r's payload lands at offset r * stride, which is exactly the
  (base, stride, nranks) form mc_decode_mean consumes in rank order 0..n-1;
* threshold (data-dependent count): counts are exchanged first, every rank
  re-packs its payload with capacity = max count, then the padded buffers are
  gathered.

Device agnostic (NCCL on CUDA tensors in production, gloo on CPU tensors in the
multi-process unit tests); world size 1 is a no-op view.
"""

from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

HDR = 32  # sizeof(mc_payload_header)


def _a16(x: int) -> int:
    return (x + 15) & ~15


def world(group=None) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def _gather_into(out: torch.Tensor, inp: torch.Tensor, group=None, async_op: bool = False):
    """all_gather_into_tensor; CUDA tensors on a gloo group are staged through host
    memory (lets several ranks share one GPU in tests — NCCL is the production path).
    With ``async_op`` (NCCL) returns the work handle; the caller's stream must ``wait()``
    on it before reading ``out``."""
    if inp.is_cuda and dist.get_backend(group) == "gloo":
        host = torch.empty(out.numel(), dtype=out.dtype)
        dist.all_gather_into_tensor(host, inp.cpu(), group=group)
        out.copy_(host)
        return None
    return dist.all_gather_into_tensor(out, inp, group=group, async_op=async_op)


def allgather_fixed(payload: torch.Tensor, out: Optional[torch.Tensor] = None, group=None,
                    async_op: bool = False):
    """Gather equal-size uint8 payload buffers; returns (gathered, stride) — or
    (gathered, stride, work) with ``async_op`` (work is None when already complete)."""
    _, n = world(group)
    stride = payload.numel()
    work = None
    if n == 1:
        out = payload
    else:
        if out is None:
            out = torch.empty(n * stride, dtype=torch.uint8, device=payload.device)
        work = _gather_into(out, payload, group, async_op=async_op)
    return (out, stride, work) if async_op else (out, stride)


def allreduce_mean_(x: torch.Tensor, group=None, async_op: bool = False):
    """Uncompressed data-parallel baseline (BASELINE config 5's comparator; reference
    ``cli._collective_for``: identity / fp16 -> allreduce, cli.py:107-109): in-place
    ``all_reduce(SUM)`` of the fp32 gradients, then ``/ f32(world)``.  The ring / NVLS
    summation order differs from ``aggregate``'s rank order for world >= 3, so it is a
    throughput comparator, not a parity target.  With ``async_op`` the
    division is left to the caller after ``work.wait()``; returns the work handle (or None)."""
    _, n = world(group)
    if n == 1:
        return None
    if x.is_cuda and dist.get_backend(group) == "gloo":  # several ranks on one GPU (tests)
        host = x.cpu()
        dist.all_reduce(host, group=group)
        x.copy_(host)
        work = None
    else:
        work = dist.all_reduce(x, group=group, async_op=async_op)
    if work is None or not async_op:
        x.div_(float(n))
        return None
    return work


def read_count(payload: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """n_idx field of the device header (u32 at byte 16) as an int64 tensor on the payload's
    device (into ``out`` when given: no allocation)."""
    v = payload[16:20].view(torch.int32)
    if out is None:
        return v.to(torch.int64)
    out.copy_(v)
    return out


def _repack(payload: torch.Tensor, count: int, cap_out: int, cap_in: Optional[int],
            out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Re-lay a sparse payload [hdr | idx[cap_in] | val[cap_in]] with capacity cap_out >= count
    (into a view of ``out`` when given: no allocation, only device copies)."""
    if cap_in is None:
        cap_in = int(payload[28:32].view(torch.int32).cpu().item())
    size = HDR + 2 * _a16(4 * cap_out)
    if out is None:
        out = torch.zeros(size, dtype=torch.uint8, device=payload.device)
    else:
        out = out[:size]
    out[:HDR].copy_(payload[:HDR])
    out[28:32].view(torch.int32).fill_(cap_out)
    out[HDR: HDR + 4 * count].copy_(payload[HDR: HDR + 4 * count])
    v_in, v_out = HDR + _a16(4 * cap_in), HDR + _a16(4 * cap_out)
    out[v_out: v_out + 4 * count].copy_(payload[v_in: v_in + 4 * count])
    return out


def allgather_variable(payload: torch.Tensor, group=None, cap_in: Optional[int] = None,
                       bufs: Optional[dict] = None) -> tuple[torch.Tensor, int, list[int]]:
    """Two-phase gather of sparse payloads with data-dependent counts (NCCL / gloo path).
    Returns (gathered, stride, counts).

    One host synchronisation per call — the padded size of the second gather is the max
    count, which the host must know to size the collective.  With ``cap_in`` (the payload's
    known capacity) and ``bufs`` (persistent ``counts`` int64[world], ``cnt`` int64[1],
    ``mine`` u8[>= payload bytes] and ``gather`` u8[>= world * payload bytes]) a step
    allocates nothing.  The zero-sync variable-size exchange is the peer push
    (GradSync.use_peer_exchange: the push kernel reads n_idx on the device)."""
    r, n = world(group)
    if n == 1:
        return payload, payload.numel(), [int(read_count(payload).item())]
    if bufs is None:
        cnt = read_count(payload)
        counts = torch.empty(n, dtype=torch.int64, device=payload.device)
    else:
        cnt = read_count(payload, bufs["cnt"])
        counts = bufs["counts"]
    _gather_into(counts, cnt.reshape(1), group)
    counts_h = [int(v) for v in counts.cpu().tolist()]  # host sync: the padded size depends on it
    cap = max(max(counts_h), 1)
    mine = _repack(payload, counts_h[r], cap, cap_in, None if bufs is None else bufs["mine"])
    if bufs is None:
        gathered, stride = allgather_fixed(mine, group=group)
    else:
        gathered, stride = allgather_fixed(mine, bufs["gather"][:n * mine.numel()], group=group)
    return gathered, stride, counts_h
