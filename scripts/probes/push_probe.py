"""encode_push into N gather buffers on this GPU (ResNet-50 set), for ncu captures / timing."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2103_15195_b200 import compressors as C, gradsets  # noqa: E402
from paper_2103_15195_b200.spec import CompressorSpec  # noqa: E402

codec, N = sys.argv[1], int(sys.argv[2])
D = sum(gradsets.sizes("resnet50_161"))
spec = CompressorSpec(codec)
x = torch.from_numpy(gradsets.synthetic_gradients("resnet50_161", 0, 0)).cuda()
res = torch.zeros(D, dtype=torch.float64, device="cuda") if spec.uses_error_feedback else None
p0 = C.device_encode(spec, x, res, None, 1)
stride = (p0.buf.numel() + 15) // 16 * 16
bufs = [torch.zeros(N * stride, dtype=torch.uint8, device="cuda") for _ in range(N)]
flg = [torch.zeros(N, dtype=torch.int32, device="cuda") for _ in range(N)]
for ep in range(1, 4):
    C.device_encode_push(spec, x, res, None, 1, bufs[0][:stride], [b.data_ptr() for b in bufs],
                         [f.data_ptr() for f in flg], ep)
    C.device_encode(spec, x, res, None, 1, out=p0.buf)
torch.cuda.synchronize()
print("ok")
