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

from .costmodel import CostParams, fit_params, microbench
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

    # ---- analytic search inputs: measured backprop profile + fitted costs
    def measure_profile(self, repetitions: int = 5) -> ModelProfile:
        """Per-tensor backward compute times on this GPU: a CUDA event is recorded on the
        backward stream when each gradient is accumulated (the same hook point that
        launches a group's sync) and the median gap to the previous one is the tensor's
        compute_time (ms).  Syncs are not armed while measuring."""
        events = {}

        def mk(i):
            def hook(_p):
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                events[i] = ev
            return hook

        hooks = [p.register_post_accumulate_grad_hook(mk(i)) for i, p in enumerate(self.params)]
        per = [[] for _ in self.params]
        try:
            for rep in range(repetitions + 1):
                self.sync.flat.zero_()
                loss = self.loss_fn(self.model)
                start = torch.cuda.Event(enable_timing=True)
                start.record()
                events.clear()
                loss.backward()
                torch.cuda.synchronize()
                if rep == 0:
                    continue  # warm-up
                prev = start
                for i in range(len(self.params)):  # backprop order = readiness order
                    ev = events.get(i)
                    if ev is None:
                        per[i].append(0.0)
                        continue
                    per[i].append(max(prev.elapsed_time(ev), 0.0))
                    prev = ev
        finally:
            for h in hooks:
                h.remove()
        import statistics

        times = [statistics.median(v) for v in per]
        return ModelProfile(type(self.model).__name__,
                            tuple(LayerProfile(i, p.numel(), t) for i, (p, t) in enumerate(zip(self.params, times))))

    def fit_costs(self, profile: Optional[ModelProfile] = None, sizes: Optional[Sequence[int]] = None,
                  repetitions: int = 10) -> CostParams:
        """CostParams from device samples: h from microbench on this GPU; g from the NCCL
        allgather of real payloads when there is more than one rank (else 0); A = the
        measured backprop time."""
        prof = profile or self.measure_profile()
        total = prof.total_size
        if sizes is None:
            sizes = sorted({max(1024, int(total * f)) for f in (0.01, 0.05, 0.1, 0.25, 0.5, 1.0)})
        h = microbench(self.sync.spec, sizes, repetitions, device=self.sync.device)
        g = ()
        if self.sync.world > 1:
            from .costmodel import comm_microbench

            g = comm_microbench(self.sync.spec, sizes, repetitions, group=self.sync.pg, device=self.sync.device)
        return fit_params(h, g, A=prof.total_compute)
