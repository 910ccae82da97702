"""Measured-time partition search with a real backward pass.

``OverlapHandle`` is the scheduler's trainer handle (``tensor_profile`` /
``timed_iteration`` / ``pin_partition``, trainer.py:325-336, 397-403) for a torch
model on one GPU rank: ``timed_iteration(partition)`` runs forward + backward with the
group syncs launched from post-accumulate-grad hooks (wait-free backprop: a group is
encoded/exchanged/decoded on the side stream while earlier layers are still in
backward) and returns the CUDA-event time of the whole iteration.  Feeding it to
``scheduler.online_search`` is MergeComp's Algorithm 2 on measured B200 iteration
times, instead of the reference's analytic simulator.
"""

from __future__ import annotations

from typing import Callable, Optional, Sequence

import torch

from .profiles import LayerProfile, ModelProfile, Partition
from .spec import CompressorSpec
from .sync import GradSync


def backprop_order(model: torch.nn.Module) -> list[torch.nn.Parameter]:
    """Trainable parameters, output layer first (reverse registration order)."""
    return [p for p in model.parameters() if p.requires_grad][::-1]


class OverlapHandle:
    def __init__(self, model: torch.nn.Module, loss_fn: Callable[[torch.nn.Module], torch.Tensor],
                 spec: CompressorSpec, root_seed: int = 0, group=None,
                 params: Optional[Sequence[torch.nn.Parameter]] = None):
        self.model = model
        self.loss_fn = loss_fn
        self.params = list(params) if params is not None else backprop_order(model)
        prof = ModelProfile.from_sizes(type(model).__name__, [p.numel() for p in self.params])
        self.sync = GradSync(spec, prof, root_seed=root_seed, group=group,
                             device=self.params[0].device)
        self.sync.attach(self.params)

    # ---- trainer-handle protocol (scheduler.online_search)
    def tensor_profile(self) -> ModelProfile:
        return self.sync.tensor_profile()

    def pin_partition(self, partition) -> None:
        self.sync.pin_partition(partition)

    def iteration(self, overlap: bool = True) -> None:
        """forward + backward + compressed sync of every group (no optimizer step)."""
        self.sync.flat.zero_()  # every .grad is a view of the fused buffer: one memset
        if overlap:
            self.sync.begin_backward()
            self.loss_fn(self.model).backward()
            self.sync.finish_backward()
        else:
            self.loss_fn(self.model).backward()
            self.sync.step()

    def timed_iteration(self, partition=None, overlap: bool = True) -> float:
        prev = self.sync.partition
        if partition is not None:
            self.sync.pin_partition(partition)
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        self.iteration(overlap)
        stop.record()
        stop.synchronize()
        ms = start.elapsed_time(stop)
        if self.sync.world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=self.sync.device)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX, group=self.sync.pg)
            ms = float(t.item())
        self.sync.pin_partition(prev)
        return ms
