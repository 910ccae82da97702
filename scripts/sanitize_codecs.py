"""Exercise every codec path once at moderate sizes, for compute-sanitizer:

    compute-sanitizer --tool memcheck python scripts/sanitize_codecs.py
    compute-sanitizer --tool racecheck python scripts/sanitize_codecs.py --small
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2103_15195_b200 import compressors as C  # noqa: E402
from paper_2103_15195_b200.spec import ALGORITHMS, CompressorSpec  # noqa: E402

small = "--small" in sys.argv
sizes = (777, 5000) if small else (777, 70_001, 300_000)
rng = np.random.default_rng(0)
for algo in ALGORITHMS:
    for kw in ({}, {"error_feedback": True, "bucket_size": 50}, {"sparsity": 0.9}):
        spec = CompressorSpec(algo, **kw)
        for n in sizes:
            x = torch.from_numpy((rng.standard_normal(n) * 1e-3).astype(np.float32)).cuda()
            st = None
            pays = []
            for w in range(2):
                p, st = C.encode(spec, x * (w + 1), st, seed=C.derive_seed(1, w, 0, 0))
                pays.append(p)
            C.aggregate(spec, pays)
            out = torch.empty_like(x)
            C.device_encode_decode(spec, x.clone(), None if st is None else st.residual,
                                   None if st is None else st.momentum, 7, out)
    torch.cuda.synchronize()
    print("ok", algo, flush=True)
