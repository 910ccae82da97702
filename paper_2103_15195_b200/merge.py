"""Merge stage of MergeComp for gradients that do NOT live in the engine's fused buffer.

The reference concatenates a partition group's per-layer gradients into one array
(``Trainer._group_slices``, trainer.py:344-348: a view of the flat host gradient).  The
sync engine keeps per-layer ``.grad`` tensors as views of one flat device buffer, so its
merge stage is zero-copy; these two calls are the copy form (K1 pack / K11 unpack of
SURVEY.md §2.1) for foreign tensors — e.g. a model whose ``.grad`` tensors were allocated by
autograd: ``mc_pack`` gathers them into a fused buffer in list order, ``mc_unpack`` scatters
the averaged result back.  Both are stream-ordered device copies (no host sync).
"""

from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch

from . import _native
from .compressors import _stream_ptr


def _check(tensors: Sequence[torch.Tensor], device) -> None:
    for t in tensors:
        if t.dtype != torch.float32 or not t.is_contiguous() or t.device != device:
            raise ValueError("merge stage: contiguous float32 tensors on the fused buffer's device only")


def pack(tensors: Sequence[torch.Tensor], fused: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Concatenate ``tensors`` (flattened, list order) into ``fused`` (allocated if None)."""
    total = sum(t.numel() for t in tensors)
    if fused is None:
        fused = torch.empty(total, dtype=torch.float32, device=tensors[0].device)
    if fused.numel() < total or fused.dtype != torch.float32:
        raise ValueError("fused buffer too small")
    _check(tensors, fused.device)
    k = len(tensors)
    ptrs = (ctypes.c_void_p * k)(*[t.data_ptr() for t in tensors])
    sizes = (ctypes.c_int64 * k)(*[t.numel() for t in tensors])
    _native.check(_native.lib().mc_pack(ptrs, sizes, k, fused.data_ptr(), _stream_ptr(stream)), "mc_pack")
    return fused


def unpack(fused: torch.Tensor, tensors: Sequence[torch.Tensor], stream=None) -> None:
    """Scatter ``fused`` back into ``tensors`` (list order) — the inverse of ``pack``."""
    total = sum(t.numel() for t in tensors)
    if fused.numel() < total or fused.dtype != torch.float32:
        raise ValueError("fused buffer too small")
    _check(tensors, fused.device)
    k = len(tensors)
    ptrs = (ctypes.c_void_p * k)(*[t.data_ptr() for t in tensors])
    sizes = (ctypes.c_int64 * k)(*[t.numel() for t in tensors])
    _native.check(_native.lib().mc_unpack(fused.data_ptr(), ptrs, sizes, k, _stream_ptr(stream)), "mc_unpack")
