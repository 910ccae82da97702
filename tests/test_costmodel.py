"""Cost model, iteration-time simulator and analytic partition search (SURVEY.md
§8(f)-2) against golden values of the reference mergesched.costmodel / simulator /
scheduler (tests/golden/make_costmodel_golden.py); CPU only, plus a GPU check that the
device-measured costs drive the analytic search end to end."""

import json
from pathlib import Path

import pytest

from paper_2103_15195_b200 import costmodel as CM, scheduler as SCH, simulator as SIM
from paper_2103_15195_b200.profiles import LayerProfile, ModelProfile, Partition
from paper_2103_15195_b200.spec import CompressorSpec

G = json.loads((Path(__file__).parent / "golden" / "costmodel.json").read_text())


def _prof(sizes, comp):
    return ModelProfile("p", tuple(LayerProfile(i, s, c) for i, (s, c) in enumerate(zip(sizes, comp))))


def _spec(algo):
    return CompressorSpec(algo, sparsity=0.999 if algo == "dgc_lite" else 0.99)


@pytest.mark.parametrize("case", range(len(G["fits"])))
def test_fit_matches_reference(case):
    c = G["fits"][case]
    f = CM.fit([CM.TimingSample(s, t, "compression") for s, t in zip(c["sizes"], c["times"])])
    assert f.B == pytest.approx(c["B"], rel=1e-9, abs=1e-12)
    assert f.gamma == pytest.approx(c["gamma"], rel=1e-9)
    assert f.residual_norm == pytest.approx(c["residual_norm"], rel=1e-6, abs=1e-12)
    assert f.intercept_clamped == c["clamped"]


def test_fit_rejects_degenerate_samples():
    with pytest.raises(ValueError):
        CM.fit([CM.TimingSample(10, 1.0, "compression")])
    with pytest.raises(ValueError):
        CM.fit([CM.TimingSample(10, 1.0, "compression"), CM.TimingSample(10, 2.0, "compression")])
    f = CM.fit([CM.TimingSample(10, 0.0, "compression"), CM.TimingSample(20, 10.0, "compression")])
    assert f.B == 0.0 and f.intercept_clamped


@pytest.mark.parametrize("case", range(len(G["sims"])))
def test_simulate_iteration_matches_reference(case):
    c = G["sims"][case]
    prof = _prof(c["sizes"], c["compute"])
    cfg = SIM.SimConfig(prof, Partition(len(c["sizes"]), tuple(c["cuts"])), _spec(c["algo"]),
                        CM.CostParams.from_dict(c["costs"]), n_workers=4, g_on_payload=c["g_on_payload"])
    got, want = SIM.simulate_iteration(cfg).to_dict(), c["report"]
    for k in ("iteration_ms", "compute_ms", "compression_ms", "communication_ms", "overlap_ms"):
        assert got[k] == pytest.approx(want[k], rel=1e-12, abs=1e-12), k
    for a, b in zip(got["per_group"], want["per_group"]):
        for k in a:
            assert a[k] == pytest.approx(b[k], rel=1e-12, abs=1e-12)


@pytest.mark.parametrize("case", range(len(G["searches"])))
def test_analytic_search_matches_reference(case):
    c = G["searches"][case]
    prof = _prof(c["sizes"], c["compute"])
    n = len(c["sizes"])
    cfg = SIM.SimConfig(prof, Partition.merged(n), _spec(c["algo"]), CM.CostParams.from_dict(c["costs"]), n_workers=4)
    res = SCH.heuristic_search(SCH.SearchConfig(Y=3, alpha=0.02, evaluator=SCH.analytic_evaluator(cfg)), prof)
    assert list(res.partition.boundaries) == c["boundaries"]
    assert res.F_ms == pytest.approx(c["F_ms"], rel=1e-12)
    assert res.termination == c["termination"]


def test_scale_comm_params_matches_reference():
    p = CM.CostParams(0.1, 1e-7, 0.2, 3e-7, 5.0)
    assert CM.scale_comm_params(p, 8, "allgather").to_dict() == pytest.approx(G["scaled_allgather_8"])
    assert CM.scale_comm_params(p, 8, "allreduce").to_dict() == pytest.approx(G["scaled_allreduce_8"])
    with pytest.raises(ValueError):
        CM.scale_comm_params(p, 8, "broadcast")


def test_cost_params_roundtrip_and_validation():
    p = CM.CostParams(0.1, 2e-7, 0.3, 4e-7, 9.0)
    assert CM.CostParams.from_dict(p.to_dict()) == p
    with pytest.raises(ValueError):
        CM.CostParams(-1.0, 0, 0, 0, 0)
    with pytest.raises(ValueError):
        CM.CostParams.from_dict({"B_h_ms": 1.0})
    with pytest.raises(ValueError):
        CM.TimingSample(0, 1.0, "compression")


@pytest.mark.gpu
def test_device_costs_drive_analytic_search():
    """microbench (CUDA events) -> fit -> analytic search on a real backward profile."""
    import torch
    torchvision = pytest.importorskip("torchvision")
    from paper_2103_15195_b200.training import OverlapHandle

    torch.manual_seed(0)
    model = torchvision.models.resnet18(weights=None).cuda()
    x = torch.randn(16, 3, 64, 64, device="cuda")
    h = OverlapHandle(model, lambda m: m(x).square().mean(), CompressorSpec("efsignsgd"))
    prof = h.measure_profile(repetitions=3)
    assert prof.n_tensors == len(h.params) and prof.total_compute > 0
    samples = CM.microbench(CompressorSpec("efsignsgd"), [1 << 16, 1 << 20, 1 << 22], 5)
    assert all(s.time > 0 for s in samples) and samples[-1].time > samples[0].time
    costs = h.fit_costs(prof, sizes=[1 << 16, 1 << 20, 1 << 22], repetitions=5)
    assert costs.gamma_h > 0 and costs.B_g == 0.0
    cfg = SIM.SimConfig(prof, Partition.merged(prof.n_tensors), CompressorSpec("efsignsgd"), costs)
    res = SCH.heuristic_search(SCH.SearchConfig(Y=3, evaluator=SCH.analytic_evaluator(cfg)), prof)
    assert res.partition.n_tensors == prof.n_tensors
    assert res.F_ms <= SIM.objective_F(cfg) + 1e-9  # never worse than the merged partition
    ms = h.timed_iteration(res.partition)
    assert ms > 0
