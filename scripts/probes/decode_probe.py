"""decode_mean of N gathered efsignsgd payloads (ResNet-50 set) in a loop, for ncu."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2103_15195_b200 import compressors as C, gradsets  # noqa: E402
from paper_2103_15195_b200.spec import CompressorSpec  # noqa: E402

codec = sys.argv[1] if len(sys.argv) > 1 else "efsignsgd"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
spec = CompressorSpec(codec)
D = sum(gradsets.sizes("resnet50_161"))
pays = []
for r in range(N):
    g = torch.from_numpy(gradsets.synthetic_gradients("resnet50_161", 0, r)).cuda()
    res = torch.zeros(D, dtype=torch.float64, device="cuda") if spec.uses_error_feedback else None
    pays.append(C.device_encode(spec, g, res, None, 1))
stride = pays[0].buf.numel()
gathered = torch.cat([p.buf for p in pays])
out = torch.empty(D, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(5):
    C.device_decode_mean(spec, gathered, stride, N, D, out, err)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    C.device_decode_mean(spec, gathered, stride, N, D, out, err)
b.record()
b.synchronize()
print(f"{codec} N={N} decode_mean {a.elapsed_time(b) / 20 * 1000:.1f} us")
