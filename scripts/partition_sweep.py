"""Partition-count sweeps of BASELINE.json configs 3 and 4 on one B200 (N = 1):

    python scripts/partition_sweep.py --gradset maskrcnn_201 --codecs randk,threshold
    python scripts/partition_sweep.py --gradset vgg16_32 --codecs topk,dgc_lite,randk,threshold,signsgd,efsignsgd,onebit,qsgd,terngrad

For every codec and y = 1..8 groups: the naive (even tensor count, scheduler.py:287-294)
partition and the analytic-optimal one for y (optimal_partition_y on the iteration model
with costs fitted on this GPU, zero compute so the objective is the pure sync time), each
timed as the device sync step (CUDA events, mean of --steps, inputs > L2).  threshold uses
tau = the 99th percentile of |g| of the set (~1% density, config 3).  Also reports the
uncompressed baseline of config 4 at this world size: the identity codec (fp32 payload;
with one rank, NCCL allreduce has nothing to exchange).  One JSON line per measurement."""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2103_15195_b200 import costmodel as CM, gradsets, simulator as SIM  # noqa: E402
from paper_2103_15195_b200.profiles import Partition  # noqa: E402
from paper_2103_15195_b200.scheduler import (SearchConfig, analytic_evaluator, heuristic_search,  # noqa: E402
                                             naive_partition, optimal_partition_y)
from paper_2103_15195_b200.spec import CompressorSpec  # noqa: E402
from paper_2103_15195_b200.sync import GradSync  # noqa: E402


def step_ms(sync, g, steps):
    for _ in range(3):
        sync.flat.copy_(g)
        sync.step()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(steps):
        sync.flat.copy_(g)  # the averaged gradient replaces the input in place: restore it
        torch.cuda.synchronize()  # (the restore is not part of the timed step)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(sync.stream)
        sync.step()
        b.record(sync.stream)
        b.synchronize()
        tot += a.elapsed_time(b)
    return tot / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gradset", default="maskrcnn_201")
    ap.add_argument("--codecs", default="randk,threshold")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--ymax", type=int, default=8)
    a = ap.parse_args()
    prof = gradsets.profile(a.gradset)
    D = prof.total_size
    gh = gradsets.synthetic_gradients(a.gradset, 0, 0)
    g = torch.from_numpy(gh).cuda()
    tau = float(np.quantile(np.abs(gh), 0.99))
    for codec in ["identity"] + a.codecs.split(","):
        kw = {"sparsity": 0.999 if codec == "dgc_lite" else 0.99}
        if codec == "threshold":
            kw["threshold"] = tau
        spec = CompressorSpec(codec, **kw)
        sizes = sorted({max(4096, int(D * f)) for f in (0.005, 0.02, 0.1, 0.3, 1.0)})
        costs = CM.fit_params(CM.microbench(spec, sizes, 5))
        cfg = SIM.SimConfig(prof, Partition.merged(prof.n_tensors), spec, costs)
        ev = analytic_evaluator(cfg)
        for y in range(1, (1 if codec == "identity" else a.ymax) + 1):
            parts = [("naive", naive_partition(prof, y))]
            if 2 <= y <= 3:  # exhaustive over the first y-2 cuts: affordable for y <= 3 only
                parts.append(("analytic_opt", optimal_partition_y(ev, prof, y)[0]))
            for kind, part in parts:
                s = GradSync(spec, prof, partition=part)
                ms = step_ms(s, g, a.steps)
                print(json.dumps({"gradset": a.gradset, "codec": codec, "y": y, "partition": kind,
                                  "boundaries": list(part.boundaries), "step_ms": round(ms, 4),
                                  "GBps": round(4 * D / ms / 1e6, 1), "predicted_ms": round(ev(part), 4),
                                  "tau": tau if codec == "threshold" else None}), flush=True)
                del s
                torch.cuda.empty_cache()
        if codec != "identity":  # MergeComp's Algorithm 2 on the analytic model, Y = ymax
            res = heuristic_search(SearchConfig(Y=a.ymax, alpha=0.02, evaluator=ev), prof)
            s = GradSync(spec, prof, partition=res.partition)
            ms = step_ms(s, g, a.steps)
            print(json.dumps({"gradset": a.gradset, "codec": codec, "y": res.partition.y, "partition": "heuristic_search",
                              "boundaries": list(res.partition.boundaries), "step_ms": round(ms, 4),
                              "GBps": round(4 * D / ms / 1e6, 1), "predicted_ms": round(res.F_ms, 4),
                              "termination": res.termination}), flush=True)
            del s
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
