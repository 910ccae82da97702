import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2103_15195_b200 import gradsets
from paper_2103_15195_b200.spec import CompressorSpec
from paper_2103_15195_b200.sync import GradSync
prof = gradsets.profile("resnet50_161")
D = prof.offsets()[-1]
s = GradSync(CompressorSpec("efsignsgd"), prof)
x = torch.from_numpy(gradsets.synthetic_gradients("resnet50_161", 0, 0)).pin_memory()
o = torch.empty(D).pin_memory()
import itertools
for wait, ch in list(itertools.product((False,), (1 << 22, 6 << 20, 1 << 23, 12 << 20, 1 << 23))) * 3:
    for _ in range(2):
        s.sync_host(x, o, wait=wait, chunk_elems=ch)
    s.sync_host_wait()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(20):
        s.sync_host(x, o, wait=wait, chunk_elems=ch)
    s.sync_host_wait()
    e1.record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"wait={wait} chunk={ch}: events {e0.elapsed_time(e1) / 20:.3f} ms/step, wall {(t1 - t0) * 1e3 / 20:.3f} ms/step")
