"""Golden values of the reference cost model / simulator / analytic search.

Run in the build container, where /root/reference exists:

    python tests/golden/make_costmodel_golden.py [/root/reference/pkg/src]

Imports ``mergesched.costmodel``, ``simulator`` and ``scheduler`` from the reference
tree and records fit results, iteration-time reports and analytic-search results on
seeded profiles into ``tests/golden/costmodel.json`` (the tests only read the JSON).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")
sys.path.insert(0, str(REF_SRC))

from mergesched import costmodel as CM, simulator as SIM, scheduler as SCH  # noqa: E402
from mergesched.compressors import CompressorSpec  # noqa: E402
from mergesched.profiles import LayerProfile, ModelProfile, Partition  # noqa: E402


def profile(seed, n):
    rng = np.random.default_rng(seed)
    sizes = [int(s) for s in rng.integers(64, 400_000, n)]
    comp = [float(c) for c in rng.uniform(0.01, 0.6, n)]
    return sizes, comp


def main():
    out = {"fits": [], "sims": [], "searches": []}
    rng = np.random.default_rng(11)
    for case in range(4):
        sizes = [int(x) for x in rng.integers(1000, 10_000_000, 6)]
        times = [float(0.02 + 3e-7 * s + rng.normal(0, 0.003)) for s in sizes]
        samples = [CM.TimingSample(size=s, time=max(t, 0.0), kind="compression") for s, t in zip(sizes, times)]
        f = CM.fit(samples)
        out["fits"].append({"sizes": sizes, "times": [max(t, 0.0) for t in times], "B": f.B, "gamma": f.gamma,
                            "residual_norm": f.residual_norm, "clamped": f.intercept_clamped})
    for seed, n, algo, cuts in ((1, 12, "efsignsgd", (3, 8)), (2, 30, "dgc_lite", (5,)), (3, 20, "qsgd", (2, 9, 15)),
                                (4, 8, "identity", ())):
        sizes, comp = profile(seed, n)
        prof = ModelProfile(name=f"p{seed}", layers=tuple(LayerProfile(i, s, c) for i, (s, c) in enumerate(zip(sizes, comp))))
        spec = CompressorSpec(algo, sparsity=0.999 if algo == "dgc_lite" else 0.99)
        costs = CM.CostParams(B_h=0.05, gamma_h=2e-7, B_g=0.03, gamma_g=1e-6, A=float(sum(comp)))
        for g_on_payload in (True, False):
            cfg = SIM.SimConfig(profile=prof, partition=Partition(n, tuple(cuts)), spec=spec, costs=costs,
                                n_workers=4, g_on_payload=g_on_payload)
            rep = SIM.simulate_iteration(cfg)
            out["sims"].append({"sizes": sizes, "compute": comp, "algo": algo, "cuts": list(cuts),
                                "costs": costs.to_dict(), "g_on_payload": g_on_payload, "report": rep.to_dict()})
        cfg = SIM.SimConfig(profile=prof, partition=Partition.merged(n) if hasattr(Partition, "merged") else Partition(n, ()),
                            spec=spec, costs=costs, n_workers=4)
        res = SCH.heuristic_search(SCH.SearchConfig(Y=3, alpha=0.02, evaluator=SCH.analytic_evaluator(cfg)), prof)
        out["searches"].append({"sizes": sizes, "compute": comp, "algo": algo, "costs": costs.to_dict(),
                                "boundaries": list(res.partition.boundaries), "F_ms": res.F_ms,
                                "termination": res.termination, "evaluations": res.evaluations})
    scaled = CM.scale_comm_params(CM.CostParams(0.1, 1e-7, 0.2, 3e-7, 5.0), 8, "allgather")
    out["scaled_allgather_8"] = scaled.to_dict()
    scaled = CM.scale_comm_params(CM.CostParams(0.1, 1e-7, 0.2, 3e-7, 5.0), 8, "allreduce")
    out["scaled_allreduce_8"] = scaled.to_dict()
    (HERE / "costmodel.json").write_text(json.dumps(out, indent=1))
    print("wrote", HERE / "costmodel.json")


if __name__ == "__main__":
    main()
