"""Exercise every codec path once at moderate sizes, for compute-sanitizer:

    compute-sanitizer --tool memcheck python scripts/sanitize_codecs.py
    compute-sanitizer --tool racecheck python scripts/sanitize_codecs.py --small

Round 2: 3- and 8-worker aggregates (table / prefetching decodes) and device-key encodes.
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
            for w in range(8 if n == sizes[-1] else 2):  # 8 workers: the 3..8-rank decode kernels
                p, st = C.encode(spec, x * (w + 1), st, seed=C.derive_seed(1, w, 0, 0))
                pays.append(p)
            C.aggregate(spec, pays[:2])
            if len(pays) > 2:
                C.aggregate(spec, pays[:3])
                C.aggregate(spec, pays)
            # graph-mode keys: the Philox key derived and read on the device
            it = torch.zeros(1, dtype=torch.int64, device="cuda")
            keys = torch.zeros(2, 2, dtype=torch.int64, device="cuda")
            C.derive_keys(1, 0, it, keys)
            C.device_encode(spec, x, None if st is None else st.residual, None if st is None else st.momentum, 0,
                            dkey=keys[0])
            out = torch.empty_like(x)
            C.device_encode_decode(spec, x.clone(), None if st is None else st.residual,
                                   None if st is None else st.momentum, 7, out)
    torch.cuda.synchronize()
    print("ok", algo, flush=True)
