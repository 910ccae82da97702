"""The data-parallel sync engine: MergeComp's per-partition compressed gradient
synchronisation on one rank (one process per GPU).

It replaces the group loop of the reference ``Trainer.step``
(trainer.py:376-389) and its timing handle (``timed_iteration`` /
``pin_partition`` / ``tensor_profile``, trainer.py:325-336, 397-403):

  merge    per-layer gradients live as views of ONE flat fp32 buffer in
           backprop order, so every partition group is a contiguous slice and
           the merge stage is zero-copy (mc_pack/mc_unpack exist for foreign
           tensors);
  encode   mc_encode on the group slice, EF residual / momentum state kept per
           (partition.boundaries, group) exactly like trainer.py:380, Philox key
           derive_seed(root, rank, iteration, group);
  exchange NCCL allgather of the aligned payload (exchange.py);
  decode   mc_decode_mean over the gathered payloads in rank order, written in
           place into the group slice (= the averaged gradient);

all on a dedicated side stream — the FIFO channel of the reference simulator
(simulator.py:114-142).  Device error flags are checked lazily (``check()``).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional, Sequence, Union

import torch

from . import _native, exchange
from .compressors import device_decode_mean, device_encode, device_encode_decode
from .profiles import LayerProfile, ModelProfile, Partition
from .spec import CompressorSpec


@dataclass
class _Chunk:
    """A bucket-aligned slice of a group with its own payload and gather buffer: the unit of
    the chunked encode -> allgather -> decode pipeline (N > 1, per-bucket codecs)."""
    start: int  # absolute element offsets in the flat buffer
    end: int
    layout: object
    payload: torch.Tensor
    gather: torch.Tensor

    @property
    def n(self) -> int:
        return self.end - self.start


@dataclass
class _Group:
    start: int
    end: int
    layout: object
    payload: torch.Tensor
    gather: Optional[torch.Tensor]
    residual: Optional[torch.Tensor]
    momentum: Optional[torch.Tensor]
    xbufs: Optional[dict] = None  # threshold over NCCL: persistent counts / re-pack buffers
    chunks: Optional[list] = None  # N > 1 chunk pipeline (GradSync.CHUNKABLE codecs)

    @property
    def n(self) -> int:
        return self.end - self.start


class GradSync:
    """Compressed gradient synchronisation for one rank.

    ``grads`` (a list of per-layer views into ``flat``) is what an autograd
    model would hold as ``.grad``; after ``step()`` they contain the
    rank-ordered mean of every rank's decoded payloads.
    """

    def __init__(
        self,
        spec: CompressorSpec,
        profile: ModelProfile,
        partition: Union[Partition, str, None] = None,
        root_seed: int = 0,
        group=None,
        device: Optional[torch.device] = None,
        stream: Optional[torch.cuda.Stream] = None,
    ):
        if not torch.cuda.is_available():
            raise _native.NativeError("GradSync needs a CUDA device (no CPU fallback)")
        _native.lib()
        self.spec = spec
        self.cspec = spec.to_c()
        self.profile = profile
        self.pg = group
        self.rank, self.world = exchange.world(group)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.stream = stream or torch.cuda.Stream(device=self.device)
        self.root_seed = int(root_seed)
        self.offsets = profile.offsets()
        self.flat = torch.zeros(self.offsets[-1], dtype=torch.float32, device=self.device)
        self.grads = [self.flat[a:b] for a, b in zip(self.offsets[:-1], self.offsets[1:])]
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.iteration = 0
        self._plans: dict[tuple, list[_Group]] = {}
        self.partition = self._resolve(partition)
        self.probe = None  # (group index, list) -> CUDA events around that group's encode
        self.fuse_local = True  # world size 1: fused encode + decode (mc_encode_decode)
        # N > 1 chunk pipeline: None = automatic (groups of >= 4M elements in ~4 chunks of
        # >= 2M), 0 = off, else the chunk length (rounded up to the bucket / word alignment)
        self.chunk_elems: Optional[int] = None
        self.sm_reserve = 16  # SMs left to NCCL while the chunk pipeline's kernels run

    # ------------------------------------------------------------ partitions / state
    def _resolve(self, partition) -> Partition:
        n = self.profile.n_tensors
        if partition is None or partition == "merged_all":
            return Partition.merged(n)
        if partition == "layer_wise":
            return Partition.layer_wise(n)
        if isinstance(partition, Partition):
            if partition.n_tensors != n:
                raise ValueError(f"partition is over {partition.n_tensors} tensors, model has {n}")
            return partition
        raise ValueError(f"unknown partition literal {partition!r}")

    def _plan(self, partition: Partition) -> list[_Group]:
        key = partition.boundaries
        plan = self._plans.get(key)
        if plan is not None:
            self._plans[key] = self._plans.pop(key)  # most recently used last
            return plan
        self._evict()
        plan = []
        ef = self.spec.uses_error_feedback
        mom = self.spec.momentum_coef is not None
        for start, end in partition.element_ranges(self.profile):
            n = end - start
            L = _native.layout(self.cspec, n)
            payload = torch.zeros(L.bytes, dtype=torch.uint8, device=self.device)
            gather = xbufs = chunks = None
            ranges = self._chunk_ranges(n)
            if ranges is not None:
                chunks = []
                for a, b in ranges:
                    Lc = _native.layout(self.cspec, b - a)
                    chunks.append(_Chunk(start + a, start + b, Lc,
                                         torch.zeros(Lc.bytes, dtype=torch.uint8, device=self.device),
                                         torch.empty(self.world * Lc.bytes, dtype=torch.uint8, device=self.device)))
            elif self.world > 1:
                gather = torch.empty(self.world * L.bytes, dtype=torch.uint8, device=self.device)
                if self.spec.algorithm == "threshold":  # padded to the step's max count, in place
                    xbufs = {"cnt": torch.zeros(1, dtype=torch.int64, device=self.device),
                             "counts": torch.zeros(self.world, dtype=torch.int64, device=self.device),
                             "mine": torch.zeros(L.bytes, dtype=torch.uint8, device=self.device),
                             "gather": gather}
            plan.append(_Group(
                start, end, L, payload, gather,
                torch.zeros(n, dtype=torch.float64, device=self.device) if ef else None,
                torch.zeros(n, dtype=torch.float32, device=self.device) if mom else None,
                xbufs, chunks,
            ))
        self._plans[key] = plan
        return plan

    # per-bucket / per-element codecs: a bucket-aligned slice encodes and decodes to exactly
    # the values of the whole group (compressors.py:291-364 work bucket by bucket).  Chunked
    # by default only where the payload is >= 1 byte per element: there the allgather costs
    # more than the encode and hiding it pays (ResNet-50, 8 ranks, projected: int8 245 -> 317,
    # fp16 171 -> 188 GB/s per GPU); for the 1-bit codecs four chunk launches on 132 SMs cost
    # more encode time than the hidden allgather saves (efsignsgd 796 -> 683 at 2 ranks)
    CHUNKABLE = frozenset({"identity", "fp16", "efsignsgd", "onebit", "int8"})
    CHUNK_AUTO = frozenset({"identity", "fp16", "int8"})
    CHUNK_MIN = 1 << 21

    def _chunk_ranges(self, n: int):
        """Relative [a, b) chunk bounds of an n-element group for the N > 1 pipeline, or None."""
        if self.world == 1 or self.chunk_elems == 0 or self.spec.algorithm not in self.CHUNKABLE:
            return None
        if getattr(self, "_dense", False) or getattr(self, "_peer", None) is not None:
            return None
        B = self.spec.bucket_size
        align = B * 32 // math.gcd(B, 32)
        if self.chunk_elems is None:
            if n < 2 * self.CHUNK_MIN or self.spec.algorithm not in self.CHUNK_AUTO:
                return None
            target = max(self.CHUNK_MIN, -(-n // 4))
        else:
            target = self.chunk_elems
        target = -(-target // align) * align
        if target >= n:
            return None
        return [(a, min(n, a + target)) for a in range(0, n, target)]

    # candidate partitions a measured search keeps alive besides the pinned one; each holds
    # an fp64 residual (8 B/elem) plus payload / gather buffers, so a Y>=3 search over
    # hundreds of candidates must not keep them all (the reference keeps every state on the
    # host, trainer.py:380; an evicted candidate restarts from zero state if revisited)
    MAX_CACHED_PLANS = 4

    def _evict(self) -> None:
        keep = {self.partition.boundaries} if hasattr(self, "partition") else set()
        graph = getattr(self, "_graph", None)
        if graph is not None:
            keep.add(graph[0])
        while len(self._plans) >= self.MAX_CACHED_PLANS + len(keep):
            victim = next((k for k in self._plans if k not in keep), None)
            if victim is None:
                break
            self._drop(victim)

    def _drop(self, key) -> None:
        self._plans.pop(key, None)
        graph = getattr(self, "_graph", None)
        if graph is not None and graph[0] == key:
            self._graph = None  # the graph holds raw pointers into the dropped buffers
        peer = getattr(self, "_peer", None)
        if peer is not None:
            for k in [k for k in peer["groups"] if k[0] == key]:
                del peer["groups"][k]

    def drop_state(self, partition: Optional[Partition] = None) -> None:
        """Free the EF/momentum state and buffers of one (or every) partition, together with
        a CUDA Graph captured over them and their peer-exchange buffers."""
        keys = list(self._plans) if partition is None else [partition.boundaries]
        for k in keys:
            self._drop(k)

    def set_gradients(self, flat: torch.Tensor) -> None:
        self.flat.copy_(flat, non_blocking=True)

    # ------------------------------------------------------------ the sync step
    def _sync_group(self, g: int, grp: _Group, dkey: Optional[torch.Tensor] = None) -> int:
        """Enqueue encode -> allgather -> decode_mean for one group; returns kernel launches.
        ``dkey``: the group's Philox key on the device (graph capture) instead of a host key."""
        seed = _native.derive_key(self.root_seed, self.rank, self.iteration, g)
        x = self.flat[grp.start:grp.end]
        probe = self.probe is not None and self.probe[0] == g
        if probe:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record(self.stream)
        key = seed[0] | (seed[1] << 64)
        if self.world == 1 and self.fuse_local:
            # single rank: aggregate([payload]) written by the encode pass itself (in place)
            device_encode_decode(self.spec, x, grp.residual, grp.momentum, key, x, payload=grp.payload, err=self.err,
                                 stream=self.stream, cspec=self.cspec, dkey=dkey)
            if probe:
                ev[1].record(self.stream)
                self.probe[1].append(ev)
            return 0
        if grp.chunks:
            pending = [self._encode_chunk(grp, c, key) for c in grp.chunks]
            if probe:
                ev[1].record(self.stream)
                self.probe[1].append(ev)
            self._decode_chunks(pending)
            return 0
        device_encode(self.spec, x, grp.residual, grp.momentum, key, out=grp.payload,
                      err=self.err, stream=self.stream, cspec=self.cspec)
        if probe:
            ev[1].record(self.stream)
            self.probe[1].append(ev)
        if self.spec.algorithm == "threshold":
            gathered, stride, _ = exchange.allgather_variable(grp.payload, group=self.pg, cap_in=grp.layout.cap,
                                                              bufs=grp.xbufs)
        else:
            gathered, stride = exchange.allgather_fixed(grp.payload, grp.gather, group=self.pg)
        device_decode_mean(self.spec, gathered, stride, self.world, grp.n, x, self.err, stream=self.stream,
                           cspec=self.cspec)
        return 0

    def _encode_chunk(self, grp: _Group, c: _Chunk, key: int):
        """Encode one chunk (state slices of its group) and start its allgather (async)."""
        a, b = c.start - grp.start, c.end - grp.start
        device_encode(self.spec, self.flat[c.start:c.end], None if grp.residual is None else grp.residual[a:b],
                      None if grp.momentum is None else grp.momentum[a:b], key, out=c.payload, err=self.err,
                      stream=self.stream, cspec=self.cspec)
        gathered, stride, work = exchange.allgather_fixed(c.payload, c.gather, group=self.pg, async_op=True)
        return c, gathered, stride, work

    def _decode_chunks(self, pending) -> None:
        for c, gathered, stride, work in pending:
            if work is not None:
                work.wait()  # the side stream waits for this chunk's gather only
            device_decode_mean(self.spec, gathered, stride, self.world, c.n, self.flat[c.start:c.end], self.err,
                               stream=self.stream, cspec=self.cspec)

    # ------------------------------------------------------------ CUDA Graph of a pinned partition
    STOCHASTIC = frozenset({"qsgd", "terngrad", "randk"})

    def capture_graph(self, partition: Optional[Partition] = None) -> None:
        """Record one rank's whole sync step for ``partition`` (default: the pinned one) as a
        CUDA Graph; ``step()`` then replays it with one launch instead of one ctypes call
        and 1-5 kernel launches per group (the launch-bound many-small-groups case of
        SURVEY.md §8(f)-4).  The stochastic codecs' Philox keys derive_seed(root, rank,
        iteration, group) are computed on the device at the head of the graph from a device
        iteration counter that every replay advances, and the encodes read them from there.

        One rank: the fused encode+decode of every group (every codec).  Several ranks with
        the peer exchange (``use_peer_exchange`` / ``try_peer_exchange``): the whole exchange
        step — encode+push of every group, then wait+decode — with the exchange epoch read
        from a device word (mc_encode_push_dev / mc_push_wait_dev) that ``step()`` rewrites
        before each replay; two graphs, one per gather-buffer parity, alternate.  The peer
        buffers are created (a collective: every rank calls this) before capturing.
        Capturing runs nothing; gradients and codec state are untouched."""
        peer = self.world > 1 and getattr(self, "_peer", None) is not None
        if not peer and (self.world != 1 or not self.fuse_local):
            raise ValueError("capture_graph: single-rank fused sync or the peer exchange only")
        from .compressors import _WS, derive_keys

        self.sync_host_wait()
        part = self.partition if partition is None else self._resolve(partition)
        self.partition = part
        plan = self._plan(part)
        need = max(max(_native.workspace_bytes(self.cspec, grp.n),
                       _native.lib().mc_decode_workspace_bytes(ctypes.byref(self.cspec), grp.n, self.world))
                   for grp in plan)
        ws = _WS.get(self.device, need, self.stream)  # sized before capture: the graph keeps these pointers
        keys = None
        if self.spec.algorithm in self.STOCHASTIC:
            self._dev_iter = torch.tensor([self.iteration], dtype=torch.int64, device=self.device)
            keys = torch.zeros(len(plan), 2, dtype=torch.int64, device=self.device)
        dep = None
        if peer:
            for g, grp in enumerate(plan):
                self._peer_group(part.boundaries, g, grp)
            dep = torch.zeros(1, dtype=torch.int32, device=self.device)
        graphs = []
        for par in ((0, 1) if peer else (None,)):
            graph = torch.cuda.CUDAGraph()
            self.stream.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.graph(graph, stream=self.stream):
                if keys is not None:
                    derive_keys(self.root_seed, self.rank, self._dev_iter, keys, stream=self.stream)
                if peer:
                    self._step_peer(plan, part.boundaries, cap=(par, dep, keys))
                else:
                    for g, grp in enumerate(plan):
                        self._sync_group(g, grp, None if keys is None else keys[g])
            graphs.append(graph)
        self._graph = (part.boundaries, graphs if peer else graphs[0], ws, len(plan), keys, dep)

    def drop_graph(self) -> None:
        self._graph = None

    # ------------------------------------------------------------ dense baseline
    def use_dense_allreduce(self) -> None:
        """Replace compress -> allgather -> decode by the uncompressed baseline of BASELINE
        config 5: per group one NCCL all_reduce(SUM) of the fp32 slice in place, then / N
        (exchange.allreduce_mean_).  The codec and its state are bypassed; groups are
        pipelined (all-reduce g+1 is issued while g's division waits)."""
        self._dense = True

    def _step_dense(self, plan) -> None:
        pending = []
        for grp in plan:
            x = self.flat[grp.start:grp.end]
            work = exchange.allreduce_mean_(x, group=self.pg, async_op=True)
            pending.append((x, work))
        for x, work in pending:
            if work is not None:
                work.wait()
                x.div_(float(self.world))

    # ------------------------------------------------------------ allgather over peer memory
    def use_peer_exchange(self, backend: str = "ipc") -> None:
        """Replace the NCCL allgather by the fused encode + push over peer memory
        (mc_encode_push / mc_push_wait): each group has two gather buffers (alternating by
        exchange epoch) and flag words that every rank maps — ``backend="ipc"`` shares them
        with CUDA IPC handles (torch.multiprocessing's reductions, exchanged over the process
        group; peer-mapped over NVLink, and also valid for several processes on one GPU),
        ``"symm"`` uses torch symmetric memory.  Each rank's encode kernel stores its payload
        straight into its slot of every rank's buffer and releases their flags when done.
        Double buffering is enough: a rank pushes epoch e+2 into the buffer a peer read at
        epoch e only after that peer's epoch-(e+1) push, which its stream issued after its
        decode of epoch e.  Threshold payloads (data-dependent count) get capacity-n slots
        and the push moves only the header and the first n_idx entries, read on the device:
        the variable-size exchange with no host round trip."""
        if self.world < 2:
            raise ValueError("the peer exchange needs more than one rank")
        if backend not in ("ipc", "symm"):
            raise ValueError(f"unknown peer backend {backend!r}")
        self._peer = {"backend": backend, "groups": {}, "epoch": 0}

    PROBE_MAGIC = 0x5EED0000

    def _all_ok(self, ok: int) -> bool:
        t = torch.tensor([ok], dtype=torch.int32, device=self.device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN, group=self.pg)
        return int(t.item()) == 1

    def try_peer_exchange(self, backend: str = "ipc") -> bool:
        """Collective probe (every rank must call it) that proves the peer path before any
        encode kernel pushes through it, else keeps the NCCL allgather:

        1. map a small probe buffer of every rank (CUDA IPC handles);
        2. enable P2P access from this device to every peer's device (mc_peer_enable —
           opening an IPC handle does not grant the importing device access);
        3. one kernel on THIS device stores ``magic | rank`` into this rank's slot of every
           rank's probe buffer (mc_peer_probe), then each rank reads back its own buffer and
           checks that every peer's store arrived.

        A step is only attempted when every rank passed the previous one (MIN all-reduce),
        so a device pair without P2P never reaches a kernel store (which would fault the
        context instead of falling back), and every collective runs on all ranks whatever
        fails locally, so a failed probe cannot deadlock."""
        if self.world < 2:
            return False
        from .compressors import _stream_ptr

        lib = _native.lib()
        self._peer = {"backend": backend, "groups": {}, "epoch": 0}
        probe = torch.zeros(self.world, dtype=torch.int32, device=self.device)
        mapped = []
        ok = 1
        try:
            if backend == "symm":
                raise RuntimeError("probe covers the IPC backend only")
            from torch.multiprocessing.reductions import reduce_tensor

            handles = [None] * self.world
            torch.cuda.synchronize(self.device)
            torch.distributed.all_gather_object(handles, reduce_tensor(probe), group=self.pg)
            for j, (fn, args) in enumerate(handles):
                mapped.append(probe if j == self.rank else fn(*args))
            for t in mapped:
                _native.check(lib.mc_peer_enable(self.device.index, t.device.index), "mc_peer_enable")
        except Exception:  # noqa: BLE001 - fall back to NCCL on every rank
            ok = 0
        if self._all_ok(ok):
            try:
                dsts = (ctypes.c_void_p * self.world)(*[t.data_ptr() + 4 * self.rank for t in mapped])
                s = torch.cuda.current_stream(self.device)
                _native.check(lib.mc_peer_probe(dsts, self.world, self.PROBE_MAGIC | self.rank, _stream_ptr(s)),
                              "mc_peer_probe")
                torch.cuda.synchronize(self.device)
            except Exception:  # noqa: BLE001
                ok = 0
            torch.distributed.barrier(group=self.pg)  # every rank's stores are complete
            if ok:
                got = [int(v) & 0xFFFFFFFF for v in probe.cpu().tolist()]
                ok = int(got == [self.PROBE_MAGIC | j for j in range(self.world)])
            if self._all_ok(ok):
                self._peer["mapped"] = mapped
                return True
        self._peer = None
        return False

    def _share(self, t: torch.Tensor) -> list[int]:
        """Device addresses of every rank's copy of ``t`` as mapped in this process."""
        if self._peer["backend"] == "symm":
            import torch.distributed._symmetric_memory as symm

            h = symm.rendezvous(t, self.pg if self.pg is not None else torch.distributed.group.WORLD)
            return [int(h.buffer_ptrs[j]) for j in range(self.world)]
        from torch.multiprocessing.reductions import reduce_tensor

        handles = [None] * self.world
        torch.distributed.all_gather_object(handles, reduce_tensor(t), group=self.pg)
        ptrs = []
        keep = self._peer.setdefault("mapped", [])
        for j, (fn, args) in enumerate(handles):
            if j == self.rank:
                ptrs.append(t.data_ptr())
            else:
                peer = fn(*args)  # opens the IPC handle: a tensor over rank j's memory
                # the handle is opened under rank j's device: grant THIS device's kernels access
                _native.check(_native.lib().mc_peer_enable(self.device.index, peer.device.index), "mc_peer_enable")
                keep.append(peer)
                ptrs.append(peer.data_ptr())
        return ptrs

    def _alloc_shared(self, numel: int, dtype) -> torch.Tensor:
        if self._peer["backend"] == "symm":
            import torch.distributed._symmetric_memory as symm

            return symm.empty(numel, dtype=dtype, device=self.device)
        return torch.empty(numel, dtype=dtype, device=self.device)

    def _peer_group(self, key, g: int, grp: _Group):
        st = self._peer["groups"].get((key, g))
        if st is None:
            stride = (grp.layout.bytes + 15) // 16 * 16
            bufs, dsts = [], []
            for _ in range(2):
                b = self._alloc_shared(self.world * stride, torch.uint8)
                b.zero_()
                ptrs = self._share(b)
                bufs.append(b)
                dsts.append([ptrs[j] + self.rank * stride for j in range(self.world)])
            fl = self._alloc_shared(2 * self.world, torch.int32)
            fl.zero_()
            torch.cuda.synchronize(self.device)
            fptrs = self._share(fl)
            flags = [[fptrs[j] + 4 * (par * self.world + self.rank) for j in range(self.world)] for par in range(2)]
            torch.distributed.barrier(group=self.pg)
            st = {"stride": stride, "bufs": bufs, "dsts": dsts, "fl": fl, "flags": flags}
            self._peer["groups"][(key, g)] = st
        return st

    def _step_peer(self, plan, key, cap=None) -> None:
        """``cap`` = (parity, device epoch word, device keys or None) while capturing a graph."""
        from .compressors import device_encode_push, device_encode_push_dev, push_wait, push_wait_dev

        if cap is None:
            self._peer["epoch"] += 1
            ep = self._peer["epoch"]
            par = ep & 1
        else:
            par, dep, keys = cap
        pend = []
        for g, grp in enumerate(plan):  # every encode pushes as it finishes: no collective launch
            st = self._peer_group(key, g, grp)
            buf = st["bufs"][par]
            own = buf[self.rank * st["stride"]:(self.rank + 1) * st["stride"]]
            x = self.flat[grp.start:grp.end]
            if cap is None:
                lo, hi = _native.derive_key(self.root_seed, self.rank, self.iteration, g)
                device_encode_push(self.spec, x, grp.residual, grp.momentum, lo | (hi << 64), own, st["dsts"][par],
                                   st["flags"][par], ep, err=self.err, stream=self.stream, cspec=self.cspec)
            else:
                device_encode_push_dev(self.spec, x, grp.residual, grp.momentum, None if keys is None else keys[g],
                                       own, st["dsts"][par], st["flags"][par], dep, self.err, stream=self.stream,
                                       cspec=self.cspec)
            pend.append((grp, st, buf))
        for grp, st, buf in pend:
            fl = st["fl"][par * self.world:(par + 1) * self.world]
            if cap is None:
                push_wait(fl, self.world, ep, err=self.err, stream=self.stream)
            else:
                push_wait_dev(fl, self.world, dep, self.err, stream=self.stream)
            device_decode_mean(self.spec, buf, st["stride"], self.world, grp.n, self.flat[grp.start:grp.end],
                               self.err, stream=self.stream, cspec=self.cspec)

    def step(self, partition: Optional[Partition] = None) -> None:
        """One synchronisation of every group of ``partition`` (default: the pinned one),
        enqueued on the side stream after the gradients' producer stream.

        With several ranks and fixed-size payloads the groups are pipelined: every
        group's encode is followed by an asynchronous allgather, and the decodes wait on
        their own gather only — encode(g+1) runs while allgather(g) is on NVLink (the
        compute and communication channels of MergeComp, simulator.py:114-142)."""
        self.sync_host_wait()
        part = self.partition if partition is None else self._resolve(partition)
        graph = getattr(self, "_graph", None)
        if graph is not None and graph[0] == part.boundaries:
            self.stream.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(self.stream):
                if graph[4] is not None:  # the graph's key schedule starts from the host iteration
                    self._dev_iter.fill_(self.iteration)  # (eager steps may have run in between)
                if graph[5] is not None:  # peer exchange: this step's epoch, the graph of its parity
                    self._peer["epoch"] += 1
                    ep = self._peer["epoch"] & 0xFFFFFFFF
                    graph[5].fill_(ep - (1 << 32) if ep >= 1 << 31 else ep)
                    graph[1][ep & 1].replay()
                else:
                    graph[1].replay()
            torch.cuda.current_stream(self.device).wait_stream(self.stream)
            self.iteration += 1
            return
        plan = self._plan(part)
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.stream):
            if getattr(self, "_dense", False):
                self._step_dense(plan)
            elif getattr(self, "_peer", None) is not None:
                self._step_peer(plan, part.boundaries)
            elif self.world > 1 and self.spec.algorithm != "threshold" and (len(plan) > 1 or plan[0].chunks):
                # every group (or chunk) is encoded and its allgather started before any
                # decode: encode(c+1) runs on the SMs while NCCL moves chunk c, decodes
                # follow in order, each waiting for its own gather only; grids leave
                # sm_reserve SMs to the NCCL kernels meanwhile
                lib = _native.lib()
                prev = lib.mc_set_sm_reserve(self.sm_reserve) if plan[0].chunks else None
                try:
                    pending = []
                    for g, grp in enumerate(plan):
                        if grp.chunks:
                            lo, hi = _native.derive_key(self.root_seed, self.rank, self.iteration, g)
                            pending += [self._encode_chunk(grp, c, lo | (hi << 64)) for c in grp.chunks]
                            continue
                        x = self._encode_group(g, grp)
                        gathered, stride, work = exchange.allgather_fixed(grp.payload, grp.gather, group=self.pg,
                                                                          async_op=True)
                        pending.append((_Chunk(grp.start, grp.end, grp.layout, grp.payload, grp.gather),
                                        gathered, stride, work))
                    self._decode_chunks(pending)
                finally:
                    if prev is not None:
                        lib.mc_set_sm_reserve(prev)
            else:
                for g, grp in enumerate(plan):
                    self._sync_group(g, grp)
        torch.cuda.current_stream(self.device).wait_stream(self.stream)
        self.iteration += 1

    def _encode_group(self, g: int, grp: _Group) -> torch.Tensor:
        lo, hi = _native.derive_key(self.root_seed, self.rank, self.iteration, g)
        x = self.flat[grp.start:grp.end]
        probe = self.probe is not None and self.probe[0] == g
        if probe:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record(self.stream)
        device_encode(self.spec, x, grp.residual, grp.momentum, lo | (hi << 64), out=grp.payload,
                      err=self.err, stream=self.stream, cspec=self.cspec)
        if probe:
            ev[1].record(self.stream)
            self.probe[1].append(ev)
        return x

    def sync_host(self, host_in: torch.Tensor, host_out: Optional[torch.Tensor] = None,
                  chunk_elems: int = 1 << 21, wait: bool = True) -> torch.Tensor:
        """The host-buffer entry point: copy a (pinned) host gradient buffer in, run one
        sync step, copy the averaged gradients back out — all stream-ordered.  On one
        rank the whole step is enqueued natively (mc_pipe_group): chunked H2D / fused
        encode+aggregate / D2H on three streams, PCIe full duplex.  ``wait=False`` leaves
        the step in flight so the next call overlaps it chunk by chunk (its H2D of a chunk
        waits only for this call's read-out of that chunk): the PCIe fill and drain of
        consecutive steps coincide.  ``sync_host_wait()`` (or any other step) joins them
        into the current stream; host_out is complete after that, and host_in must not be
        rewritten before it (its H2D copies may still be in flight)."""
        if host_out is None:
            host_out = torch.empty(self.flat.numel(), dtype=torch.float32, pin_memory=True)
        if self.world == 1 and self.fuse_local and chunk_elems > 0:
            return self._sync_host_native(host_in, host_out, chunk_elems, wait)
        self.sync_host_wait()
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.stream):
            self.flat.copy_(host_in, non_blocking=True)
        self.step()
        with torch.cuda.stream(self.stream):
            host_out.copy_(self.flat, non_blocking=True)
        torch.cuda.current_stream(self.device).wait_stream(self.stream)  # host_out is ready in stream order
        return host_out

    def sync_host_wait(self) -> None:
        """Make the current stream wait for every sync_host(wait=False) step in flight."""
        if getattr(self, "_pipe_pending", False):
            from .compressors import _stream_ptr

            _native.check(_native.lib().mc_pipe_finish(self._pipe, _stream_ptr(self.stream), _stream_ptr(self._d2h),
                                                       _stream_ptr(torch.cuda.current_stream(self.device))),
                          "mc_pipe_finish")
            self._pipe_pending = False

    def _sync_host_native(self, host_in, host_out, chunk_elems, wait=True):
        import ctypes

        from .compressors import _WS, _stream_ptr

        lib = _native.lib()
        if getattr(self, "_pipe", None) is None:
            h = ctypes.c_void_p()
            _native.check(lib.mc_pipe_create(ctypes.byref(h)), "mc_pipe_create")
            self._pipe = h
            self._h2d = torch.cuda.Stream(device=self.device)
            self._d2h = torch.cuda.Stream(device=self.device)
        if not (host_in.is_pinned() and host_out.is_pinned()):
            raise ValueError("sync_host needs pinned host buffers")
        cur = torch.cuda.current_stream(self.device)
        for st in (self._h2d, self.stream, self._d2h):
            st.wait_stream(cur)
        plan = self._plan(self.partition)
        sh, se, sd = _stream_ptr(self._h2d), _stream_ptr(self.stream), _stream_ptr(self._d2h)
        for g, grp in enumerate(plan):
            lo, hi = _native.derive_key(self.root_seed, self.rank, self.iteration, g)
            ws = _WS.get(self.device, _native.workspace_bytes(self.cspec, grp.n), self.stream)
            _native.check(lib.mc_pipe_group(
                self._pipe, ctypes.byref(self.cspec), host_in.data_ptr() + 4 * grp.start,
                host_out.data_ptr() + 4 * grp.start, self.flat.data_ptr() + 4 * grp.start, grp.n, chunk_elems,
                None if grp.residual is None else grp.residual.data_ptr(),
                None if grp.momentum is None else grp.momentum.data_ptr(), lo, hi, grp.payload.data_ptr(),
                ws.data_ptr(), ws.numel(), self.err.data_ptr(), sh, se, sd), "mc_pipe_group")
        _native.check(lib.mc_pipe_finish(self._pipe, se, sd, _stream_ptr(cur) if wait else _native.MC_PIPE_NO_WAIT),
                      "mc_pipe_finish")
        self._pipe_pending = not wait
        self.iteration += 1
        return host_out

    def __del__(self):
        pipe = getattr(self, "_pipe", None)
        if pipe is not None:
            try:
                _native.lib().mc_pipe_destroy(pipe)
            except Exception:
                pass

    # ------------------------------------------------------------ overlap with backward (WFBP)
    def attach(self, params_backprop_order: Sequence[torch.nn.Parameter]) -> None:
        """Bind model parameters (listed in backprop-readiness order, i.e. the profile's
        order) to the fused buffer: every ``p.grad`` becomes a view of ``flat``, and a
        post-accumulate-grad hook launches a group's sync on the side stream as soon as
        its last tensor is ready — the reference simulator's FIFO channel
        ``start_i = max(finish_{i-1}, ready_i)`` (simulator.py:114-142) on real hardware.
        Zero gradients with ``zero_grad(set_to_none=False)`` so the views persist."""
        params = list(params_backprop_order)
        if [p.numel() for p in params] != self.profile.sizes():
            raise ValueError("parameters do not match the profile sizes (backprop order)")
        for p, g in zip(params, self.grads):
            if p.device != self.device or p.dtype != torch.float32:
                raise ValueError("GradSync.attach needs fp32 parameters on the sync device")
            p.grad = g.view_as(p)
        self._params = params
        self._hooks = [p.register_post_accumulate_grad_hook(self._make_hook(i)) for i, p in enumerate(params)]
        self._armed = False

    def _make_hook(self, i: int):
        def hook(_p):
            if self._armed:
                self._tensor_ready(i)
        return hook

    def begin_backward(self) -> None:
        """Arm the hooks for one backward pass under the pinned partition."""
        self.sync_host_wait()
        plan = self._plan(self.partition)
        ranges = self.partition.group_ranges()
        self._group_of = [g for g, (a, b) in enumerate(ranges) for _ in range(a, b)]
        self._left = [b - a for a, b in ranges]
        self._next_group = 0
        self._launched = [False] * len(plan)
        self._armed = True

    def _tensor_ready(self, i: int) -> None:
        g = self._group_of[i]
        self._left[g] -= 1
        # groups go out in order (one FIFO channel): launch every consecutive complete group
        while self._next_group < len(self._left) and self._left[self._next_group] == 0:
            self._launch_group(self._next_group)
            self._next_group += 1

    def _launch_group(self, g: int) -> None:
        grp = self._plan(self.partition)[g]
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(self.device))  # the backward stream produced it
        self.stream.wait_event(ready)
        with torch.cuda.stream(self.stream):
            self._sync_group(g, grp)
        self._launched[g] = True

    def finish_backward(self) -> None:
        """Launch any group not triggered yet (e.g. tensors without gradients) and make the
        caller's stream wait for the averaged gradients; advances the iteration."""
        if not self._armed:
            raise RuntimeError("finish_backward() without begin_backward()")
        for g in range(len(self._launched)):
            if not self._launched[g]:
                self._launch_group(g)
        torch.cuda.current_stream(self.device).wait_stream(self.stream)
        self._armed = False
        self.iteration += 1

    def detach(self) -> None:
        for h in getattr(self, "_hooks", []):
            h.remove()
        self._hooks = []

    def check(self) -> None:
        """Raise the reference's ValueError if any device error flag was set.

        Non-finite gradients: the reference raises before touching codec state
        (compressors.py:384-385); the engine's kernels consume a group in one in-place pass,
        so the steps since the last check() may have folded the non-finite values into the
        EF residual / momentum.  Rather than carry NaN forever, the state of every cached
        partition is reset to zeros (the codec memory at t = 0) before raising — a skipped
        (e.g. AMP overflow) step costs the EF memory, not the run."""
        self.sync_host_wait()
        flags = int(self.err.item())
        if flags:
            self.err.zero_()
            from .compressors import _raise_flags

            if flags & _native.MC_ERR_NONFINITE:
                for plan in self._plans.values():
                    for grp in plan:
                        if grp.residual is not None:
                            grp.residual.zero_()
                        if grp.momentum is not None:
                            grp.momentum.zero_()
            _raise_flags(flags)

    # ------------------------------------------------------------ scheduler handle
    def tensor_profile(self) -> ModelProfile:
        """trainer.py:325-333 — sizes in backprop order (compute times unknown)."""
        return ModelProfile(self.profile.name, tuple(LayerProfile(i, l.size, 0.0) for i, l in enumerate(self.profile.layers)))

    def pin_partition(self, partition) -> None:
        self.partition = self._resolve(partition)

    def timed_iteration(self, partition: Union[Partition, str, None] = None) -> float:
        """Device time (ms) of one sync step under ``partition`` — CUDA events on the
        side stream, max over ranks (trainer.py:397-403 uses wall time)."""
        part = self.partition if partition is None else self._resolve(partition)
        self._plan(part)
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        start.record(self.stream)
        self.step(part)
        stop.record(self.stream)
        stop.synchronize()
        ms = start.elapsed_time(stop)
        if self.world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=self.device)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX, group=self.pg)
            ms = float(t.item())
        return ms
