"""Sync-step time of many-group partitions, eager (one ctypes call + 1-5 launches per
group) vs a CUDA Graph of the pinned partition (GradSync.capture_graph), one B200, N=1.
One JSON line per (codec, partition)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2103_15195_b200 import gradsets  # noqa: E402
from paper_2103_15195_b200.profiles import Partition  # noqa: E402
from paper_2103_15195_b200.scheduler import naive_partition  # noqa: E402
from paper_2103_15195_b200.spec import CompressorSpec  # noqa: E402
from paper_2103_15195_b200.sync import GradSync  # noqa: E402


def timed(sync, reps=50):
    for _ in range(5):
        sync.step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        sync.step()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    prof = gradsets.profile("resnet50_161")
    g = torch.from_numpy(gradsets.synthetic_gradients("resnet50_161", 0, 0)).cuda()
    for codec in ("efsignsgd", "dgc_lite", "signsgd", "qsgd", "randk"):
        spec = CompressorSpec(codec, sparsity=0.99 if codec == "randk" else 0.999)
        for name, part in (("naive_y8", naive_partition(prof.n_tensors, 8)),
                           ("naive_y32", naive_partition(prof.n_tensors, 32)),
                           ("layer_wise", Partition.layer_wise(prof.n_tensors))):
            s = GradSync(spec, prof, partition=part)
            s.flat.copy_(g)
            eager = timed(s)
            s.capture_graph()
            graph = timed(s)
            print(json.dumps({"codec": codec, "partition": name, "groups": part.y, "eager_ms": round(eager, 4),
                              "graph_ms": round(graph, 4), "speedup": round(eager / graph, 2)}), flush=True)


if __name__ == "__main__":
    main()
