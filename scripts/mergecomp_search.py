"""MergeComp on B200 with a real model: measured-time partition search (Algorithm 2,
online_search with Y=2) where each candidate is timed as a full forward + backward
with the compressed group syncs overlapped with backward (WFBP hooks).

    python scripts/mergecomp_search.py [--model resnet50] [--codec efsignsgd] [--batch 64]

Prints iteration times for merged / layer-wise / naive-even / searched partitions and
the sequential (no overlap) baseline, one JSON line.  Random-init weights, synthetic
batch (no datasets offline)."""

import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2103_15195_b200.profiles import Partition  # noqa: E402
from paper_2103_15195_b200.scheduler import SearchConfig, naive_partition, online_search  # noqa: E402
from paper_2103_15195_b200.spec import CompressorSpec  # noqa: E402
from paper_2103_15195_b200.training import OverlapHandle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--codec", default="efsignsgd")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--res", type=int, default=224)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torchvision

    torch.backends.cudnn.benchmark = True
    model = getattr(torchvision.models, a.model)(weights=None).cuda()
    x = torch.randn(a.batch, 3, a.res, a.res, device="cuda")
    y = torch.randint(0, 1000, (a.batch,), device="cuda")
    loss_fn = lambda m: torch.nn.functional.cross_entropy(m(x), y)  # noqa: E731
    spec = CompressorSpec(a.codec, sparsity=0.999 if a.codec in ("topk", "dgc_lite") else 0.99)
    h = OverlapHandle(model, loss_fn, spec)
    n = h.tensor_profile().n_tensors

    def med(part, overlap=True):
        for _ in range(3):
            h.timed_iteration(part, overlap)
        return statistics.median(h.timed_iteration(part, overlap) for _ in range(a.reps))

    res = {"model": a.model, "codec": a.codec, "batch": a.batch, "tensors": n}
    res["merged_ms"] = med(Partition.merged(n))
    res["merged_sequential_ms"] = med(Partition.merged(n), overlap=False)
    res["layerwise_ms"] = med(Partition.layer_wise(n))
    res["naive_y2_ms"] = med(naive_partition(n, 2))
    search = online_search(SearchConfig(Y=2, alpha=0.02), h, repetitions=a.reps)
    res["searched"] = {"boundaries": list(search.partition.boundaries), "F_ms": search.F_ms,
                       "evaluations": search.evaluations, "termination": search.termination}
    res["searched_ms"] = med(search.partition)
    # analytic search: measured backprop profile + device-fitted costs,
    # Algorithm 2 on the iteration-time model, no timed iterations per candidate
    import time as _time

    from paper_2103_15195_b200 import simulator as SIM
    from paper_2103_15195_b200.scheduler import analytic_evaluator, heuristic_search

    t0 = _time.perf_counter()
    prof = h.measure_profile(repetitions=5)
    costs = h.fit_costs(prof, repetitions=10)
    cfg = SIM.SimConfig(prof, Partition.merged(n), spec, costs)
    ares = heuristic_search(SearchConfig(Y=2, alpha=0.02, evaluator=analytic_evaluator(cfg)), prof)
    res["analytic"] = {"costs": costs.to_dict(), "boundaries": list(ares.partition.boundaries),
                       "predicted_F_ms": ares.F_ms, "evaluations": ares.evaluations,
                       "predicted_merged_ms": SIM.objective_F(cfg), "search_wall_s": _time.perf_counter() - t0,
                       "measured_ms": med(ares.partition)}
    fwd_bwd = []
    for _ in range(a.reps):  # compute-only reference: forward + backward, no sync
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        h.sync.flat.zero_()
        loss_fn(model).backward()
        e.record()
        e.synchronize()
        fwd_bwd.append(s.elapsed_time(e))
    res["forward_backward_only_ms"] = statistics.median(fwd_bwd)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
