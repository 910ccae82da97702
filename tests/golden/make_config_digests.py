"""SHA-256 digests of the REAL reference's outputs on the BASELINE.json configs at full size.

Run in the build container, where /root/reference exists (the GPU box never reads it):

    python tests/golden/make_config_digests.py [--only CASE ...] [--jobs 6]

For every case it regenerates the SURVEY.md §8(d) synthetic gradients
(``gradsets.synthetic_gradients``: per-tensor N(0, sigma_t^2), numpy
default_rng(1000*iteration + rank), one all-zero tensor), drives the group loop of
the reference ``Trainer.step`` (trainer.py:376-389: per group, per worker
``encode(spec, g[sl], state[(boundaries, w, g)], seed=derive_seed(root, w, t, g))``,
then ``aggregate``) with ``mergesched.compressors`` itself, and records digests of
every payload section, the fp64 residual, the fp32 momentum and the aggregated mean
per (iteration, worker, group), plus the digest of every input gradient so the GPU
test can prove it regenerated the same bits.  Written to ``tests/golden/configs.json``
(digests keep the repository small; the GPU test ``tests/test_gpu_configs.py``
recomputes the same quantities on the B200 and compares).

Top-k / DGC: the tie set at the k-th magnitude is recorded per encode.  numpy's
argpartition tie choice is implementation-defined; a case whose
boundary tie straddles the selection is flagged ``straddle`` and its digests after
that point are not comparable (the GPU keeps the lowest indices).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF_SRC = Path("/root/reference/pkg/src")
OUT = HERE / "configs.json"


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(f"{a.dtype.str}:{a.size}:".encode())
    h.update(a.tobytes())
    return h.hexdigest()[:32]


def cut_at(sizes, target):
    """Tensor boundary whose element offset is closest to ``target`` (SURVEY.md §8(a) Y=2 cuts)."""
    off = np.cumsum([0] + list(sizes))
    return int(np.argmin(np.abs(off[1:-1] - target)) + 1)


def cases() -> list[dict]:
    sys.path.insert(0, str(ROOT))
    from paper_2103_15195_b200 import gradsets

    r50, r101 = gradsets.sizes("resnet50_161"), gradsets.sizes("resnet101_314")
    mrc, vgg = gradsets.sizes("maskrcnn_201"), gradsets.sizes("vgg16_32")
    out = []

    def add(cid, gradset, spec, bounds, workers, iters, root, cfg):
        out.append(dict(cid=cid, gradset=gradset, spec=spec, boundaries=list(bounds), workers=workers,
                        iters=iters, root=root, config=cfg))

    # config 1: R50, dgc_lite 0.999 + EF, Partition(161, (160,)), 1 worker, 3 iterations
    add("c1_dgc_r50", "resnet50_161", {"algorithm": "dgc_lite", "sparsity": 0.999}, (160,), 1, 3, 101, 1)
    # config 2: R50 efsignsgd / onebit (bucket 512, EF on), the Y=2 cut of the reference search, 8 ranks
    b2 = cut_at(r50, 25_506_408)
    for algo in ("efsignsgd", "onebit"):
        add(f"c2_{algo}_r50_w8", "resnet50_161", {"algorithm": algo}, (b2,), 8, 3, 102, 2)
    # config 3: R101 qsgd 8-bit / terngrad (EF off), the qsgd n=8 cut, 8 ranks
    b3 = cut_at(r101, 35_743_208)
    add("c3_qsgd_r101_w8", "resnet101_314", {"algorithm": "qsgd", "levels": 256, "bucket_size": 512}, (b3,), 8, 2, 103, 3)
    add("c3_terngrad_r101_w8", "resnet101_314", {"algorithm": "terngrad"}, (b3,), 8, 2, 103, 3)
    # config 4: Mask R-CNN randk 1% and threshold tau = p99(|g|), naive partitions y = 1..8, 2 ranks
    g0 = gradsets.synthetic_gradients("maskrcnn_201", 0, 0)
    tau = float(np.percentile(np.abs(g0), 99))
    for y in range(1, 9):
        bounds = _naive(len(mrc), y)
        add(f"c4_randk_mrcnn_y{y}", "maskrcnn_201", {"algorithm": "randk", "sparsity": 0.99}, bounds, 2, 2, 104, 4)
        add(f"c4_threshold_mrcnn_y{y}", "maskrcnn_201", {"algorithm": "threshold", "threshold": tau}, bounds, 2, 2,
            104, 4)
    # config 5: VGG-16, the nine north-star codecs + the four secondary ones, naive y=2, 2 ranks x 2 iterations
    bv = _naive(len(vgg), 2)
    for algo in ("topk", "dgc_lite", "randk", "threshold", "signsgd", "efsignsgd", "onebit", "qsgd", "terngrad",
                 "fp16", "int8", "signum", "identity"):
        spec = {"algorithm": algo}
        if algo == "dgc_lite":
            spec["sparsity"] = 0.999
        add(f"c5_{algo}_vgg16", "vgg16_32", spec, bv, 2, 2, 105, 5)
    del r50, r101
    return out


def _naive(n, y):
    base, rem = divmod(n, y)
    counts = [base + 1] * rem + [base] * (y - rem)
    return tuple(int(v) for v in np.cumsum(counts)[:-1])


def _tie_info(R, spec, work32, k):
    mag = np.abs(work32)
    n = len(mag)
    if k >= n:
        return None
    kth = np.partition(mag, n - k)[n - k]
    greater = int((mag > kth).sum())
    equal = int((mag == kth).sum())
    info = {"kth": float(kth), "greater": greater, "equal": equal, "straddle": greater + equal > k}
    if info["straddle"]:  # the strictly-greater set and the tie set, for the §9.1 contract check
        info["greater_idx"] = sha(np.flatnonzero(mag > kth).astype(np.uint32))
        info["tie_idx"] = [int(i) for i in np.flatnonzero(mag == kth)]
    return info


def run_case(c: dict) -> dict:
    sys.path.insert(0, str(REF_SRC))
    sys.path.insert(0, str(ROOT))
    from mergesched import compressors as R  # the reference itself

    from paper_2103_15195_b200 import gradsets

    t0 = time.time()
    spec = R.CompressorSpec(**c["spec"])
    sizes = gradsets.sizes(c["gradset"])
    off = np.cumsum([0] + list(sizes))
    cuts = [0] + c["boundaries"] + [len(sizes)]
    slices = [(int(off[a]), int(off[b])) for a, b in zip(cuts[:-1], cuts[1:])]
    states = {}
    rec = {"inputs": {}, "steps": []}
    for t in range(c["iters"]):
        grads = []
        for w in range(c["workers"]):
            g = gradsets.synthetic_gradients(c["gradset"], t, w)
            rec["inputs"][f"t{t}.w{w}"] = sha(g)
            grads.append(g)
        for gi, (a, b) in enumerate(slices):
            payloads = []
            step = {"t": t, "g": gi, "workers": []}
            for w in range(c["workers"]):
                x = grads[w][a:b]
                st = states.get((w, gi))
                ent = {}
                if spec.algorithm in ("topk", "dgc_lite"):
                    work = x.astype(np.float64)
                    if st is not None and spec.uses_error_feedback:
                        work = work + st.residual
                    ent["tie"] = _tie_info(R, spec, work.astype(np.float32), R.top_k_count(spec.sparsity, b - a))
                seed = R.derive_seed(c["root"], w, t, gi)
                p, st = R.encode(spec, x, st, seed=seed)
                states[(w, gi)] = st
                if ent.get("tie") and ent["tie"]["straddle"]:
                    ent["tie"]["ref_tie_picks"] = sorted(set(ent["tie"]["tie_idx"]) & set(int(i) for i in p.indices))
                payloads.append(p)
                ent["idx"] = None if p.indices is None else sha(np.asarray(p.indices, np.uint32))
                ent["n_idx"] = 0 if p.indices is None else int(len(p.indices))
                ent["val"] = sha(np.asarray(p.values, np.float32))
                ent["bits"] = None if p.bits is None else sha(np.asarray(p.bits, np.uint8))
                ent["flags"] = int(p.flags)
                ent["res"] = None if st is None or not spec.uses_error_feedback else sha(st.residual)
                ent["mom"] = None if st is None or st.momentum is None else sha(st.momentum)
                step["workers"].append(ent)
            mean = R.aggregate(spec, payloads)
            step["mean"] = sha(np.asarray(mean, np.float32))
            rec["steps"].append(step)
    rec["seconds"] = round(time.time() - t0, 1)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--jobs", type=int, default=6)
    a = ap.parse_args()
    todo = [c for c in cases() if not a.only or c["cid"] in a.only]
    old = json.loads(OUT.read_text()) if OUT.exists() and a.only else {"cases": []}
    keep = [c for c in old["cases"] if c["cid"] not in {t["cid"] for t in todo}]
    # heaviest first (VGG-16, then R101)
    order = sorted(todo, key=lambda c: {"vgg16_32": 0, "resnet101_314": 1}.get(c["gradset"], 2))
    with ProcessPoolExecutor(a.jobs) as ex:
        results = list(ex.map(run_case, order))
    for c, r in zip(order, results):
        c.update(r)
        ties = [w["tie"] for s in r["steps"] for w in s["workers"] if w.get("tie")]
        flag = " STRADDLE" if any(tt["straddle"] for tt in ties) else ""
        print(f"{c['cid']}: {r['seconds']} s{flag}", flush=True)
    allc = sorted(keep + order, key=lambda c: c["cid"])
    import platform

    OUT.write_text(json.dumps({"numpy": np.__version__, "machine": platform.machine(),
                               "generator": "tests/golden/make_config_digests.py", "reference": "mergesched (pkg/src)",
                               "cases": allc}, indent=1))
    print(f"wrote {OUT} ({len(allc)} cases)")


if __name__ == "__main__":
    main()
