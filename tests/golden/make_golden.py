"""Generate golden vectors by running the REAL reference package (mergesched).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py [/root/reference/pkg/src]

It imports ``mergesched.compressors`` from the reference tree, drives the
per-group sync loop of ``Trainer.step`` (trainer.py:377-389: encode per worker
with per-(worker, group) state and derive_seed(root, w, t, g) keys, then
aggregate) on seeded inputs, and records inputs, payload sections, residual /
momentum states and the aggregated means into ``tests/golden/codecs.npz``.
The GPU box never reads /root/reference; the tests only read the .npz.

Every top-k case is checked to be tie-free at the k-th boundary so that the
reference's implementation-defined argpartition tie choice cannot matter.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")
sys.path.insert(0, str(REF_SRC))

from mergesched import compressors as R  # noqa: E402  (the reference itself)

sys.path.insert(0, str(HERE))
from inputs import case_inputs, x_digest  # noqa: E402


def _tie_free(x_corr, k):
    mag = np.abs(x_corr)
    if k >= len(mag):
        return True
    kth = np.sort(mag)[::-1][k - 1]
    nxt = np.sort(mag)[::-1][k]
    return kth != nxt


CASES = []


def case(cid, spec_kw, n, workers=1, iters=1, root=5, style="normal"):
    CASES.append(dict(cid=cid, spec=spec_kw, n=n, workers=workers, iters=iters, root=root, style=style))


LENGTHS = (1, 7, 63, 300, 512, 1000, 4109)
for algo in R.ALGORITHMS:
    for n in LENGTHS:
        case(f"{algo}_n{n}", {"algorithm": algo}, n, workers=1, iters=2, root=11)
    # EF forced on for every codec, 3 workers x 3 iterations (SURVEY §4 EF decomposition)
    kw = {"algorithm": algo, "error_feedback": True, "sparsity": 0.9}
    case(f"{algo}_ef_w3", kw, 777, workers=3, iters=3, root=21)
    case(f"{algo}_zeros_w2", {"algorithm": algo, "error_feedback": False}, 2100, workers=2, iters=1, root=31, style="zeros")

# parameter variants
case("topk_s05", {"algorithm": "topk", "sparsity": 0.5, "error_feedback": False}, 4, root=1)
case("topk_s999_big", {"algorithm": "topk", "sparsity": 0.999}, 40_003, workers=2, iters=2, root=3)
case("dgc_s999_big", {"algorithm": "dgc_lite", "sparsity": 0.999}, 30_001, workers=1, iters=3, root=4)
case("dgc_mom", {"algorithm": "dgc_lite", "sparsity": 0.9, "momentum": 0.9}, 5000, workers=2, iters=3, root=6)
case("signum_mom", {"algorithm": "signum"}, 5000, workers=2, iters=3, root=7)
case("signum_mom05_ef", {"algorithm": "signum", "momentum": 0.5, "error_feedback": True}, 3001, workers=2, iters=3, root=8)
case("signsgd_big", {"algorithm": "signsgd"}, 40_017, workers=2, iters=1, root=9)
case("qsgd_l16_b64", {"algorithm": "qsgd", "levels": 16, "bucket_size": 64}, 3000, workers=2, iters=2, root=12, style="zeros")
case("qsgd_l5_b50", {"algorithm": "qsgd", "levels": 5, "bucket_size": 50}, 1234, workers=2, iters=2, root=13)
case("qsgd_l2", {"algorithm": "qsgd", "levels": 2, "bucket_size": 32}, 999, workers=1, iters=2, root=14)
case("qsgd_l1000", {"algorithm": "qsgd", "levels": 1000, "bucket_size": 128}, 2049, workers=2, iters=1, root=15)
case("qsgd_big", {"algorithm": "qsgd"}, 33_600, workers=2, iters=2, root=16, style="zeros")
case("terngrad_b64", {"algorithm": "terngrad", "bucket_size": 64}, 3001, workers=2, iters=2, root=17, style="zeros")
case("terngrad_big", {"algorithm": "terngrad"}, 33_600, workers=2, iters=1, root=18, style="zeros")
case("efsign_b32", {"algorithm": "efsignsgd", "bucket_size": 32}, 1000, workers=2, iters=3, root=19)
case("efsign_b50", {"algorithm": "efsignsgd", "bucket_size": 50}, 1000, workers=2, iters=3, root=20)
case("efsign_b1000", {"algorithm": "efsignsgd", "bucket_size": 1000}, 5003, workers=2, iters=2, root=22)
case("efsign_big", {"algorithm": "efsignsgd"}, 33_151, workers=2, iters=2, root=23)
case("onebit_b50", {"algorithm": "onebit", "bucket_size": 50}, 1000, workers=2, iters=3, root=24, style="zeros")
case("onebit_big", {"algorithm": "onebit"}, 33_151, workers=2, iters=2, root=25)
case("onebit_b2048", {"algorithm": "onebit", "bucket_size": 2048}, 9000, workers=2, iters=2, root=26)
case("int8_b256", {"algorithm": "int8", "bucket_size": 256}, 1000, workers=2, iters=1, root=27, style="zeros")
case("int8_b7", {"algorithm": "int8", "bucket_size": 7}, 1000, workers=2, iters=1, root=28)
case("randk_floyd", {"algorithm": "randk", "sparsity": 0.99}, 44_454, workers=2, iters=1, root=29)
case("randk_small_n", {"algorithm": "randk", "sparsity": 0.5, "unbiased_scaling": True}, 5000, workers=2, iters=2, root=2)
case("randk_tail_shuffle", {"algorithm": "randk", "sparsity": 0.9}, 20_000, workers=2, iters=1, root=30)
case("randk_full", {"algorithm": "randk", "sparsity": 0.0}, 64, workers=1, iters=1, root=32)
case("threshold_tau05", {"algorithm": "threshold", "threshold": 0.5}, 5000, workers=3, iters=2, root=33)
case("threshold_none", {"algorithm": "threshold", "threshold": 99.0}, 100, workers=2, iters=1, root=34)
case("threshold_ef", {"algorithm": "threshold", "threshold": 1.0, "error_feedback": True}, 3000, workers=2, iters=3, root=35)
case("fp16_range", {"algorithm": "fp16"}, 4000, workers=2, iters=1, root=36)
case("topk_dyadic_ef", {"algorithm": "topk", "sparsity": 0.75}, 64, workers=1, iters=3, root=37, style="dyadic")


def run_case(c, store):
    spec = R.CompressorSpec(**c["spec"])
    xs = case_inputs(c)
    states = [None] * c["workers"]
    pre = c["cid"]
    for t in range(c["iters"]):
        payloads = []
        for w in range(c["workers"]):
            x = xs[t][w]
            seed = R.derive_seed(c["root"], w, t, 0)
            if spec.algorithm in ("topk", "dgc_lite"):
                # tie-free guard on the corrected buffer the codec will see
                corr = x.astype(np.float64)
                if states[w] is not None:
                    base = states[w].momentum if spec.momentum_coef is not None else None
                    work = x if base is None else (np.float32(spec.momentum_coef) * base + x)
                    corr = work + states[w].residual
                k = R.top_k_count(spec.sparsity, c["n"])
                assert _tie_free(corr.astype(np.float32), k) or c["style"] == "dyadic", c["cid"]
            p, s = R.encode(spec, x, states[w], seed=seed)
            states[w] = s
            payloads.append(p)
            key = f"{pre}.t{t}.w{w}"
            if c["n"] <= 1000:
                store[key + ".x"] = x
            store[key + ".xdigest"] = np.array([x_digest(x)], np.uint64)
            store[key + ".seed"] = np.array([seed & (2 ** 64 - 1), seed >> 64], np.uint64)
            if p.indices is not None:
                store[key + ".idx"] = p.indices
            store[key + ".val"] = p.values
            if p.bits is not None:
                store[key + ".bits"] = p.bits
            store[key + ".flags"] = np.array([p.flags], np.int64)
            if c["n"] <= 1100:
                store[key + ".ser"] = np.frombuffer(R.serialize(p), np.uint8)
                store[key + ".dec"] = R.decode(spec, p)
            if s is not None and (c["n"] <= 5000 or t == c["iters"] - 1):
                store[key + ".res"] = s.residual
                if s.momentum is not None:
                    store[key + ".mom"] = s.momentum
        store[f"{pre}.t{t}.mean"] = R.aggregate(spec, payloads)


def main():
    store = {}
    meta = []
    for c in CASES:
        run_case(c, store)
        meta.append(c)
    # derive_seed table and pairwise means
    seeds = []
    for root in (0, 1, 7, 2 ** 32 + 5, 2 ** 63 + 11):
        for w in (0, 3):
            for t in (0, 1, 999):
                for g in (0, 1, 7):
                    s = R.derive_seed(root, w, t, g)
                    seeds.append([root & (2**64 - 1), w, t, g, s & (2 ** 64 - 1), s >> 64])
    store["derive_seed.table"] = np.array(seeds, np.uint64)
    rng = np.random.default_rng(99)
    lens = [1, 5, 8, 9, 127, 128, 129, 255, 256, 300, 511, 512, 513, 1000, 4096, 65537]
    for n in lens:
        a = np.abs(rng.standard_normal(n).astype(np.float32))
        store[f"mean.n{n}.a"] = a
        store[f"mean.n{n}.m"] = np.array([a.mean()], np.float32)
    store["mean.lengths"] = np.array(lens, np.int64)
    np.savez_compressed(HERE / "codecs.npz", **store)
    (HERE / "codecs.json").write_text(json.dumps({"numpy": np.__version__, "cases": meta}, indent=1))
    print(f"wrote {len(store)} arrays, {len(meta)} cases")


if __name__ == "__main__":
    main()
