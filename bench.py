"""Benchmark: fp32 gradient GB/s through compress -> allgather -> decompress (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--codec efsignsgd] [--gradset resnet50_161]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...      # the CPU reference arm (oracle port, host cores)

Workload (BASELINE.json configs[1]): the ResNet-50 gradient set (161 tensors,
25,557,032 fp32) with EFSignSGD (bucket 512, error feedback, bit-packing),
MergeComp partition search enabled (online_search, Y=2, alpha=0.02, on measured
GPU sync times), one sync step = every group: encode -> NCCL allgather ->
decode + rank-ordered mean written in place into the gradients.  The per-GPU
work is fixed as N grows (weak scaling); value = N * 4 * D / T_step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fp32 gradient GB/s through compress→allgather→decompress at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--codec", default="efsignsgd")
    ap.add_argument("--gradset", default="resnet50_161")
    ap.add_argument("--sparsity", type=float, default=None)
    ap.add_argument("--no-search", action="store_true", help="skip the partition search (merged partition)")
    ap.add_argument("--boundaries", default=None, help="comma separated cut list instead of the search")
    ap.add_argument("--search-reps", type=int, default=20)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--e2e-chunk", type=int, default=1 << 23,
                    help="elements per pipelined H2D/encode/D2H chunk (8M: 32 MB copies, measured best once "
                         "consecutive steps overlap; scripts/probes/e2e_debug.py)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "p2p", "nccl", "allreduce_dense"],
                    help="N > 1: fused encode + push over NVLink peer memory (falls back to NCCL if the "
                         "peer mapping fails on any rank), the NCCL allgather, or auto: the push where the "
                         "payload is >= 1/8 of the fp32 gradient (byte codecs, where overlapping the exchange "
                         "with the encode pays; profiles/r1_projection_multi_gpu.jsonl), NCCL for the 1-bit "
                         "and sparse codecs; allreduce_dense: the uncompressed fp32 NCCL all_reduce + /N "
                         "baseline of BASELINE config 5 (codec ignored)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--step-mode", default="auto", choices=["auto", "graph", "eager"],
                    help="graph: time CUDA Graph replays of the pinned step (GradSync.capture_graph: one rank, or "
                         "the peer exchange) after the eager pass that feeds the roofline probes; auto = graph "
                         "where the step is capturable, else eager")
    ap.add_argument("--graph", action="store_const", const="graph", dest="step_mode", help="= --step-mode graph")
    ap.add_argument("--eager", action="store_const", const="eager", dest="step_mode", help="= --step-mode eager")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="bounded CPU oracle sample budget")
    ap.add_argument("--json-out", default=None)
    return ap.parse_args()


def spec_for(args):
    from paper_2103_15195_b200.spec import CompressorSpec

    kw = {}
    if args.sparsity is not None:
        kw["sparsity"] = args.sparsity
    elif args.codec in ("topk", "dgc_lite"):
        kw["sparsity"] = 0.999
    return CompressorSpec(args.codec, **kw)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks (NVML, sampled during the timed region)
class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self.period = period_s
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - clocks are reported as unavailable
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv:
            self._t.join()

    def summary(self):
        if not self.nv or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        names = [k for k, v in self.REASONS.items() if self.reasons & v and k != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ------------------------------------------------------------------ host placement + PCIe probe (e2e context)
def numa_bind(device_index: int):
    """Pin this process to the CPUs of the GPU's NUMA node (read from sysfs) before the
    pinned host buffers are allocated and first touched, so the e2e copies do not cross the
    socket interconnect.  Returns {"node", "cpus"} or None where sysfs has no answer."""
    try:
        import torch

        pr = torch.cuda.get_device_properties(device_index)
        bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        node = int(Path(f"/sys/bus/pci/devices/{bdf}/numa_node").read_text().strip())
        if node < 0:
            return {"node": node, "cpus": None, "bdf": bdf}
        cpus = set()
        for part in Path(f"/sys/devices/system/node/node{node}/cpulist").read_text().strip().split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
        return {"node": node, "cpus": len(cpus), "bdf": bdf}
    except Exception:  # noqa: BLE001 - placement is best effort, reported as unknown
        return None


def pcie_probe(host_in, host_out, dev, reps: int = 10):
    """Same-run bound of the e2e leg: the step's H2D of ``host_in`` and D2H into ``host_out``
    (pinned, the e2e's own buffers) issued together on two streams — PCIe full duplex.
    Returns GB/s of fp32 gradient (bytes of one direction / time), CUDA events."""
    import torch

    n = host_in.numel()
    da = torch.empty(n, dtype=torch.float32, device=dev)
    db = torch.zeros(n, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    cur = torch.cuda.current_stream(dev)

    def one():
        for st in (s1, s2):
            st.wait_stream(cur)
        with torch.cuda.stream(s1):
            da.copy_(host_in, non_blocking=True)
        with torch.cuda.stream(s2):
            host_out.copy_(db, non_blocking=True)
        for st in (s1, s2):
            cur.wait_stream(st)

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        for _ in range(reps):
            fn()
        b.record(cur)
        torch.cuda.synchronize(dev)
        return a.elapsed_time(b) / reps

    def h2d():
        da.copy_(host_in, non_blocking=True)

    def d2h():
        host_out.copy_(db, non_blocking=True)

    B = 4.0 * n
    r = {"duplex_GBps": B / timed(one) / 1e6, "h2d_GBps": B / timed(h2d) / 1e6, "d2h_GBps": B / timed(d2h) / 1e6}
    del da, db
    return r


# ------------------------------------------------------------------ CPU oracle timing
def cpu_oracle_rate(spec, gradset: str, workers: int, budget_s: float, partition=None, cores: int = 1):
    """Time the numpy oracle (reference semantics) on the same workload: the
    per-group encode of every simulated worker then aggregate (trainer.py:376-389).
    Runs whole sync steps of the full gradient set until ~budget_s elapsed (>= 1 step).
    Returns (GB/s, seconds, steps)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import numpy as np

    import mergecomp_oracle as O
    from paper_2103_15195_b200 import gradsets
    from paper_2103_15195_b200.profiles import Partition

    prof = gradsets.profile(gradset)
    part = partition or Partition.merged(prof.n_tensors)
    ranges = part.element_ranges(prof)
    grads = [gradsets.synthetic_gradients(gradset, 0, w) for w in range(workers)]
    states = {}
    D = prof.total_size
    t0 = time.perf_counter()
    steps = 0
    while True:
        for g, (a, b) in enumerate(ranges):
            pays = []
            for w in range(workers):
                p, states[(g, w)] = O.encode(spec, grads[w][a:b], states.get((g, w)), seed=O.derive_seed(0, w, steps, g))
                pays.append(p)
            O.aggregate(spec, pays)
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return workers * 4.0 * D * steps / el / 1e9, el, steps


_REF_FLAT = None  # the sample buffer, inherited by the forked workers (no pickling of data)


def _oracle_chunk(args):
    """Worker-process body of the reference arm: one bucket-aligned chunk of _REF_FLAT."""
    spec_doc, lo, hi, workers, seed_base = args
    sys.path.insert(0, str(ROOT / "oracle"))
    import mergecomp_oracle as O
    from paper_2103_15195_b200.spec import CompressorSpec

    spec = CompressorSpec(**spec_doc)
    x = _REF_FLAT[lo:hi]
    pays = [O.encode(spec, x, None, seed=O.derive_seed(seed_base, w, 0, 0))[0] for w in range(workers)]
    O.aggregate(spec, pays)
    return hi - lo


def run_reference(args):
    """--impl reference: the reference's CPU path (the oracle port — the reference is
    pure numpy and cannot travel to the GPU box) on the same metric/config, on all
    host cores via one process per core, each step a bounded bucket-aligned sample."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp

    import numpy as np

    from paper_2103_15195_b200 import gradsets

    global _REF_FLAT
    spec = spec_for(args)
    cores = os.cpu_count() or 1
    n_workers = max(1, args.gpus)
    flat = _REF_FLAT = gradsets.synthetic_gradients(args.gradset, 0, 0)
    D = flat.size
    B = spec.bucket_size
    budget_total = 150.0
    total_steps = args.steps + args.warmup
    per_step_budget = budget_total / max(total_steps, 1)
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        def one_step(sample):
            chunk = max(B, (sample // cores) // B * B)
            jobs = []
            off = 0
            while off < sample:
                jobs.append((spec.to_dict(), off, min(off + chunk, sample), n_workers, 0))
                off += chunk
            t0 = time.perf_counter()
            done = sum(pool.map(_oracle_chunk, jobs))
            return done, time.perf_counter() - t0

        sample = min(D, 512 * 1024 * cores)
        _, t_probe = one_step(sample)
        rate = sample / max(t_probe, 1e-6)
        sample = int(min(D, max(4096 * cores, rate * per_step_budget)))
        for _ in range(args.warmup):
            one_step(sample)
        times, elems = [], 0
        for _ in range(args.steps):
            e, t = one_step(sample)
            times.append(t)
            elems += e
        total = sum(times)
    value = n_workers * 4.0 * elems / total / 1e9
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{args.gradset} {spec.algorithm} (oracle port of mergesched, numpy)",
                   "codec": spec.to_dict(), "sample_elements_per_step": sample, "simulated_workers": n_workers},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"{sample} of {D} elements per step, bucket-aligned chunks over {cores} processes"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2103_15195_b200 import _native, gradsets
    from paper_2103_15195_b200.profiles import Partition
    from paper_2103_15195_b200.scheduler import SearchConfig, online_search
    from paper_2103_15195_b200.sync import GradSync

    rank, world, local = dist_env()
    assert world == args.gpus or world == 1, f"WORLD_SIZE={world} but --gpus {args.gpus}"
    # one process per GPU; MC_BENCH_BACKEND=gloo lets several ranks share one GPU (payloads
    # staged through host memory) to exercise the multi-rank flow where only one GPU exists
    backend = os.environ.get("MC_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    placement = numa_bind(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    spec = spec_for(args)
    prof = gradsets.profile(args.gradset)
    D = prof.total_size

    dense = args.exchange == "allreduce_dense"
    if dense:
        from paper_2103_15195_b200.spec import CompressorSpec

        spec = CompressorSpec("identity")
        args.no_search = args.no_search or not args.boundaries
    sync = GradSync(spec, prof, root_seed=0, device=dev)
    exchange_used = "none (one rank)"
    if dense:
        sync.use_dense_allreduce()
        exchange_used = "uncompressed fp32 NCCL all_reduce(SUM) + /N per group (config 5 comparator)"
    elif world > 1:
        exchange_used = "nccl allgather"
        from paper_2103_15195_b200.spec import payload_bytes

        want_p2p = args.exchange == "p2p" or (args.exchange == "auto" and payload_bytes(spec, D) * 8 >= 4 * D)
        if want_p2p and sync.try_peer_exchange():
            exchange_used = "encode fused with push over peer memory (CUDA IPC, NVLink)"
    host_grads = torch.from_numpy(gradsets.synthetic_gradients(args.gradset, 0, rank)).pin_memory()
    sync.flat.copy_(host_grads)
    torch.cuda.synchronize()

    # ---- partition: MergeComp online search on measured GPU sync times (Algorithm 2)
    search = None
    if args.boundaries:
        sync.pin_partition(Partition(prof.n_tensors, tuple(int(b) for b in args.boundaries.split(","))))
    elif not args.no_search:
        for _ in range(5):
            sync.step()
        search = online_search(SearchConfig(Y=2, alpha=0.02), sync, repetitions=args.search_reps)
        sync.drop_state()  # fresh EF state for the pinned partition
        sync.pin_partition(search.partition)
    part = sync.partition
    sizes = part.group_sizes(prof)
    sync.flat.copy_(host_grads)

    # ---- probes: events around the dominant kernel (largest group's encode) on the sync stream
    big = max(range(len(sizes)), key=lambda i: sizes[i])
    probes = []
    sync.probe = (big, probes)

    for _ in range(max(args.warmup, 3)):
        sync.step()
    torch.cuda.synchronize()
    sync.check()
    probes.clear()

    lib = _native.lib()
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = lib.mc_kernel_launches()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    with sampler:
        start.record(sync.stream)
        for _ in range(args.steps):
            sync.step()
        stop.record(sync.stream)
        torch.cuda.synchronize()
    launches = lib.mc_kernel_launches() - l0
    ms = start.elapsed_time(stop)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    torch.cuda.synchronize()
    sync.check()
    ms_step = ms / args.steps
    step_mode = "eager (one C-ABI call per group per step)"
    step_modes = None
    capturable = sync.world == 1 or getattr(sync, "_peer", None) is not None
    if args.step_mode == "graph" or (args.step_mode == "auto" and capturable):
        # the same step as one CUDA Graph replay: the same kernels (launches counted in the eager
        # pass above), no per-launch host gaps; inputs still the previous step's output (in place)
        sync.probe = None
        sync.capture_graph()
        for _ in range(max(args.warmup, 3)):
            sync.step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        gsampler = ClockSampler(local)  # clocks of the graph-timed region
        with gsampler:
            start.record(sync.stream)
            for _ in range(args.steps):
                sync.step()
            stop.record(sync.stream)
            torch.cuda.synchronize()
        ms = start.elapsed_time(stop)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        sync.check()
        sync.drop_graph()
        graph_ms_step = ms / args.steps
        step_modes = {"eager_ms_per_step": ms_step, "graph_ms_per_step": graph_ms_step}
        # auto reports the faster of the two (the stochastic codecs' graphs read device-derived
        # Philox keys instead of host-expanded constant-bank round keys, which can cost more
        # than the launches they save); --graph reports the graph
        if args.step_mode == "graph" or graph_ms_step < ms_step:
            ms_step = graph_ms_step
            step_mode = "CUDA Graph replay of the pinned step"
            sampler = gsampler
    value = world * 4.0 * D / (ms_step * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (EF bucket encode of the largest group)
    kern_ms = statistics.mean(a.elapsed_time(b) for a, b in probes) if probes else None
    L = _native.layout(spec.to_c(), sizes[big])
    n_big = sizes[big]
    ef = 16 if spec.uses_error_feedback else 0
    mom = 8 if spec.momentum_coef is not None else 0
    fused = world == 1 and spec.algorithm in ("efsignsgd", "onebit", "int8", "qsgd", "terngrad")
    # read g, r/w fp64 residual, write own payload (+ write the averaged gradient when fused at N=1)
    alg_bytes = n_big * (4 + ef + mom + (4 if fused else 0)) + (L.bytes - 32)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9 if kern_ms else None
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(f"{spec.algorithm}:{n_big}")
    sync.probe = None

    # ---- end to end through the public API: pinned host gradients in, averaged gradients out
    out_host = torch.empty(D, dtype=torch.float32).pin_memory()
    for _ in range(2):
        sync.sync_host(host_grads, out_host, chunk_elems=args.e2e_chunk)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()  # every sync_host stream waits on the current stream, so this precedes all copies
    for _ in range(args.e2e_steps):
        # each step copies its gradient in and its result out; consecutive steps overlap chunk
        # by chunk (step t+1's H2D of a chunk waits for step t's read-out of it)
        sync.sync_host(host_grads, out_host, chunk_elems=args.e2e_chunk, wait=False)
    sync.sync_host_wait()
    e1.record()  # the current stream now waits on every step's D2H and encode
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = world * 4.0 * D / (e2e_ms / args.e2e_steps * 1e-3) / 1e9
    pcie = pcie_probe(host_grads, out_host, dev)  # same buffers, same run: what bounds e2e here

    # ---- CPU baseline: the oracle on this host, rank 0 at N=1 only, bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, secs, steps = cpu_oracle_rate(spec, args.gradset, 1, args.cpu_seconds, part)
        cpu = {"value": rate, "unit": "GB/s", "cores": 1, "kind": "port",
               "sample": f"{steps} full sync step(s) of {args.gradset} ({D} fp32), partition {list(part.boundaries)}, "
                         f"1 worker, numpy single thread, {secs:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": {
                "workload": f"{args.gradset} ({prof.n_tensors} tensors, {D} fp32) {spec.algorithm} "
                            f"bucket {spec.bucket_size}{' +EF' if spec.uses_error_feedback else ''}, "
                            f"MergeComp partition {'search (Y=2)' if search else 'fixed'}",
                "codec": spec.to_dict(),
                "partition": list(part.boundaries),
                "group_sizes": sizes,
                "search": None if search is None else {"evaluations": search.evaluations,
                                                       "termination": search.termination, "F_ms": search.F_ms},
                "parallelism": f"dp{world}",
                "exchange": exchange_used,
                "l2": "inputs larger than L2 (grads 4D + fp64 residual 8D bytes per rank, >> 126 MB)",
                "input": "step t+1 encodes the averaged gradient written by step t (in place)",
                "step_mode": step_mode,
                "step_modes_ms": step_modes,
            },
            "roofline": {
                "bound": "hbm",
                "kernel": ("k_bucket_pipe (fused encode+decode, N=1)" if fused else "encode kernel") + " of the largest group",
                "achieved": achieved,
                "peak": peak,
                "unit": "GB/s",
                "frac": None if achieved is None else achieved / peak,
                "traffic": traffic,
                "algorithmic_bytes_per_launch": alg_bytes,
                "kernel_ms": kern_ms,
                "kernel_share_of_step": None if kern_ms is None else kern_ms / ms_step,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback 6650 GB/s",
                "kernel_timing": "CUDA events around the kernel on the sync stream in the eager pass (the event "
                                 "records add ~2-3 us); in graph mode the replayed step bounds the kernel from above",
            },
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": 4 * D, "d2h_bytes_per_step": 4 * D,
                    "ms_per_step": e2e_ms / args.e2e_steps,
                    "pcie": pcie, "pcie_frac": e2e_value / world / pcie["duplex_GBps"],
                    "host_placement": placement},
            "gpu_launches": int(launches),
            "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)
        if args.json_out:
            Path(args.json_out).write_text(json.dumps(line, indent=1))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
