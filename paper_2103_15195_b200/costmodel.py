"""Affine cost model fitted from B200 measurements.

API mirror of the reference ``mergesched.costmodel`` (costmodel.py:1-188): a sync
of x elements costs ``h(x) = B_h + gamma_h x`` for compression (encode + decode +
EF update) and ``g(x) = B_g + gamma_g x`` for the exchange, both in ms, fitted by
least squares.  What changes is where the samples come from: ``microbench`` times
the sm_100a encode + rank-mean decode with CUDA events on the device (the
reference times numpy with ``perf_counter``), and ``comm_microbench`` times the
NCCL allgather of real payload sizes; with those, ``scheduler.analytic_evaluator``
searches partitions without running 20 iterations per candidate.
"""

from __future__ import annotations

import statistics
from dataclasses import dataclass
from typing import Iterable, NamedTuple, Optional, Sequence

import numpy as np
import torch

from .spec import CompressorSpec

_KINDS = ("compression", "communication")


@dataclass(frozen=True)
class CostParams:
    """Fitted costs in ms (slopes in ms / element); ``A`` = backprop compute per iteration
    (costmodel.py:22-60)."""

    B_h: float
    gamma_h: float
    B_g: float
    gamma_g: float
    A: float

    def __post_init__(self):
        for k in ("B_h", "gamma_h", "B_g", "gamma_g", "A"):
            if getattr(self, k) < 0:
                raise ValueError(f"{k} must be >= 0, got {getattr(self, k)}")

    def to_dict(self) -> dict:
        return {"B_h_ms": self.B_h, "gamma_h_ms_per_elem": self.gamma_h, "B_g_ms": self.B_g,
                "gamma_g_ms_per_elem": self.gamma_g, "A_ms": self.A}

    @classmethod
    def from_dict(cls, doc: dict) -> "CostParams":
        keys = ("B_h_ms", "gamma_h_ms_per_elem", "B_g_ms", "gamma_g_ms_per_elem", "A_ms")
        missing = [k for k in keys if k not in doc]
        if missing:
            raise ValueError(f"cost params document missing key {missing[0]!r}")
        return cls(*(float(doc[k]) for k in keys))


@dataclass(frozen=True)
class TimingSample:
    """One (elements, ms) point of either kind (costmodel.py:63-78)."""

    size: int
    time: float
    kind: str

    def __post_init__(self):
        if self.size < 1:
            raise ValueError(f"sample size must be >= 1, got {self.size}")
        if self.time < 0:
            raise ValueError(f"sample time must be >= 0, got {self.time}")
        if self.kind not in _KINDS:
            raise ValueError(f"sample kind must be compression|communication, got {self.kind!r}")


def h_cost(params: CostParams, x: float) -> float:
    if x < 0:
        raise ValueError("x must be >= 0")
    return params.B_h + params.gamma_h * x


def g_cost(params: CostParams, x: float) -> float:
    if x < 0:
        raise ValueError("x must be >= 0")
    return params.B_g + params.gamma_g * x


class FitResult(NamedTuple):
    B: float
    gamma: float
    residual_norm: float
    intercept_clamped: bool


def fit(samples: Sequence[TimingSample]) -> FitResult:
    """Ordinary least squares of time on size; a negative intercept is clamped to 0 and
    flagged (costmodel.py:102-121)."""
    if len(samples) < 2:
        raise ValueError("need at least 2 samples to fit a line")
    x = np.array([s.size for s in samples], dtype=np.float64)
    y = np.array([s.time for s in samples], dtype=np.float64)
    if np.all(x == x[0]):
        raise ValueError("all sample sizes are equal; the slope is unidentifiable")
    gamma, b = np.polyfit(x, y, 1)
    clamped = bool(b < 0)
    b = max(float(b), 0.0)
    return FitResult(b, float(gamma), float(np.linalg.norm(y - (b + gamma * x))), clamped)


def _event_median(fn, repetitions: int, warmup: int, stream: torch.cuda.Stream, batch: int = 8) -> float:
    """Median over ``repetitions`` of the mean device time of ``batch`` back-to-back calls
    (CUDA events on the launch stream).  A spin kernel ahead of the start event keeps the
    GPU busy while the host enqueues the batch, so host launch overhead never appears as
    idle time between the events: the samples are kernel time only."""
    for _ in range(warmup):
        fn()
    times = []
    for _ in range(repetitions):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            torch.cuda._sleep(2_000_000)  # ~1 ms at 1.9 GHz: covers the enqueue of the batch
        a.record(stream)
        for _ in range(batch):
            fn()
        b.record(stream)
        b.synchronize()
        times.append(a.elapsed_time(b) / batch)
    return statistics.median(times)


def microbench(spec: CompressorSpec, sizes: Iterable[int], repetitions: int, seed: int = 0, warmup: int = 2,
               device: Optional[torch.device] = None) -> list[TimingSample]:
    """Device time of one compression pass per size: encode (with the EF / momentum
    update) + the rank-mean decode of the payload, CUDA events on the launch stream,
    median of ``repetitions`` after ``warmup`` (costmodel.py:124-154)."""
    from . import compressors as C

    if repetitions < 3:
        raise ValueError(f"repetitions must be >= 3, got {repetitions}")
    dev = device or torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    gen = torch.Generator(device=dev).manual_seed(seed)
    out = []
    for n in sizes:
        n = int(n)
        g = torch.randn(n, generator=gen, device=dev) * 1e-3
        res = torch.zeros(n, dtype=torch.float64, device=dev) if spec.uses_error_feedback else None
        mom = torch.zeros(n, device=dev) if spec.momentum_coef is not None else None
        pay = C.device_encode(spec, g, res, mom, seed)
        dec = torch.empty(n, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)

        def once():
            C.device_encode(spec, g, res, mom, seed, out=pay.buf)
            C.device_decode_mean(spec, pay.buf, pay.buf.numel(), 1, n, dec, err)

        out.append(TimingSample(n, _event_median(once, repetitions, warmup, stream), "compression"))
    return out


def comm_microbench(spec: CompressorSpec, sizes: Iterable[int], repetitions: int, group=None, warmup: int = 2,
                    device: Optional[torch.device] = None) -> list[TimingSample]:
    """Device time of the NCCL allgather of one group's payload (payload_bytes(spec, x)
    per rank), max over ranks.  Needs an initialised process group with > 1 rank."""
    import torch.distributed as dist

    from .exchange import allgather_fixed
    from .spec import payload_bytes

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) < 2:
        raise ValueError("comm_microbench needs a process group with at least 2 ranks")
    dev = device or torch.device("cuda", torch.cuda.current_device())
    world = dist.get_world_size(group)
    stream = torch.cuda.current_stream(dev)
    out = []
    for n in sizes:
        pb = (payload_bytes(spec, int(n)) + 15) // 16 * 16
        buf = torch.zeros(pb, dtype=torch.uint8, device=dev)
        gathered = torch.empty(world * pb, dtype=torch.uint8, device=dev)
        t = _event_median(lambda: allgather_fixed(buf, gathered, group=group), repetitions, warmup, stream)
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX, group=group)
        out.append(TimingSample(int(n), float(tt.item()), "communication"))
    return out


def scale_comm_params(params: CostParams, n_workers: int, collective: str, reference_workers: int = 2) -> CostParams:
    """Rescale (B_g, gamma_g) from the calibration worker count: ring allreduce moves
    ~2(n-1)/n per element, allgather of payloads ~(n-1) (costmodel.py:157-188)."""
    if n_workers < 1:
        raise ValueError("n_workers must be >= 1")
    if reference_workers < 2:
        raise ValueError("reference_workers must be >= 2")
    vol = {"allreduce": lambda n: 2.0 * (n - 1) / n, "allgather": lambda n: float(n - 1)}.get(collective)
    if vol is None:
        raise ValueError(f"collective must be allreduce|allgather, got {collective!r}")
    f = vol(n_workers) / vol(reference_workers)
    return CostParams(params.B_h, params.gamma_h, params.B_g * f, params.gamma_g * f, params.A)


def fit_params(compression: Sequence[TimingSample], communication: Sequence[TimingSample] = (),
               A: float = 0.0) -> CostParams:
    """CostParams from samples of both kinds; without communication samples (one rank)
    the exchange costs nothing."""
    h = fit(compression)
    if communication:
        g = fit(communication)
        return CostParams(h.B, max(h.gamma, 0.0), g.B, max(g.gamma, 0.0), A)
    return CostParams(h.B, max(h.gamma, 0.0), 0.0, 0.0, A)
