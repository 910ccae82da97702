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
