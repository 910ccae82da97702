"""One decode_mean over N stacked payloads of the ResNet-50 set (for ncu captures)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2103_15195_b200 import compressors as C, gradsets  # noqa: E402
from paper_2103_15195_b200.spec import CompressorSpec  # noqa: E402

codec, N = sys.argv[1], int(sys.argv[2])
gs = sys.argv[3] if len(sys.argv) > 3 else "resnet50_161"
D = sum(gradsets.sizes(gs))
spec = CompressorSpec(codec)
res = (lambda: torch.zeros(D, dtype=torch.float64, device="cuda")) if spec.uses_error_feedback else (lambda: None)
pays = [C.device_encode(spec, torch.from_numpy(gradsets.synthetic_gradients(gs, 0, r)).cuda(), res(), None, 1)
        for r in range(N)]
stride = pays[0].buf.numel()
gathered = torch.cat([p.buf for p in pays])
out = torch.empty(D, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    C.device_decode_mean(spec, gathered, stride, N, D, out, err)
torch.cuda.synchronize()
print("ok", int(err.item()))
if "--time" in sys.argv:
    import time  # noqa: F401
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        torch.cuda._sleep(5_000_000)
        s.record()
        for _ in range(50):
            C.device_decode_mean(spec, gathered, stride, N, D, out, err)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 50)
    print(f"{codec} N={N} decode_mean {best * 1e3:.1f} us")
