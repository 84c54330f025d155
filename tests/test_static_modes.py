"""Static provisioning baselines (ls/provisioner.py:516-561) on the device vs the reference's
own PlanScorer(mode='staratio'|'stapsratio') records (tests/golden/make_static_goldens.py)."""
import numpy as np
import pytest

from goldens import inline_instance, instance, plans_array, plan_from_str, read_jsonl
from paper_2111_10635_b200.errors import InvariantError
from paper_2111_10635_b200.model import SchedulingPlan
from paper_2111_10635_b200.scoring import PlanScorer

ITEMS = read_jsonl("static.jsonl.gz")


def _inst(it):
    return instance(it["instance"]) if "instance" in it else inline_instance(it)


def test_static_goldens_cover_both_modes_and_outcomes():
    modes = {it["mode"] for it in ITEMS}
    assert modes == {"staratio", "stapsratio"}
    st = [r["status"] for it in ITEMS for r in it["records"]]
    assert st.count(0) > 1000 and st.count(10) > 1000 and st.count(255) > 0
    # stapsratio charges cpu_per_gpu PS cores per accelerator unit (ls/provisioner.py:545)
    assert any(r.get("ps", 0) > 0 for it in ITEMS if it["mode"] == "stapsratio" for r in it["records"])
    assert all(r.get("ps", 0) == 0 for it in ITEMS if it["mode"] == "staratio" for r in it["records"])


def test_unknown_mode_raises_like_reference():
    g, c, job = instance("cfg1")
    with pytest.raises(InvariantError):
        PlanScorer(g, c, job, mode="bogus")


@pytest.mark.gpu
def test_device_static_modes_match_reference():
    torch = pytest.importorskip("torch")
    for it in ITEMS:
        g, c, job = _inst(it)
        recs = it["records"]
        sc = PlanScorer(g, c, job, mode=it["mode"])
        out = sc.score_arrays(plans_array(recs))
        torch.cuda.synchronize()
        h = {k: v.cpu().numpy() for k, v in out.items() if v is not None}
        code = h["status"].astype(np.int64) & 0x7F
        for i, r in enumerate(recs):
            if r["status"] == 255:
                assert code[i] == 8, (it["mode"], r["plan"])
                continue
            assert code[i] == r["status"], (it["mode"], r["plan"], int(code[i]), r["status"])
            assert np.float64(h["cost"][i]).view(np.int64) == np.float64(float.fromhex(r["cost"])).view(np.int64)
            if r["status"] == 0:
                S = int(h["num_stages"][i])
                assert h["k"][i, :S].tolist() == r["k"], (r["plan"], h["k"][i, :S].tolist(), r["k"])
                assert int(h["ps"][i]) == r["ps"]
            else:
                assert h["gap"][i] == 1.0


@pytest.mark.gpu
def test_static_scorer_objects_and_provision_api():
    from paper_2111_10635_b200.errors import InfeasibleError
    from paper_2111_10635_b200.scoring import provision, static_provision
    it = next(x for x in ITEMS if x.get("instance") == "cfg2" and x["mode"] == "stapsratio")
    g, c, job = _inst(it)
    sc = PlanScorer(g, c, job, mode="stapsratio")
    ok = [r for r in it["records"] if r["status"] == 0][:20]
    bad = [r for r in it["records"] if r["status"] == 10][:20]
    for r in ok:
        plan = SchedulingPlan(tuple(plan_from_str(r["plan"])))
        s = sc(plan)
        assert s.feasible and s.cost == float.fromhex(r["cost"])
        assert list(s.provisioning.per_stage_k) == r["k"] and s.provisioning.ps_cores == r["ps"]
        assert sorted([t, n] for t, n in s.provisioning.per_type_totals.items()) == sorted(r["totals"])
        assert s.report.monetary_cost == s.cost
        p = provision(plan, g, c, job, mode="stapsratio")
        assert p == static_provision(plan, g, c, job, "stapsratio") == s.provisioning
    for r in bad:
        plan = SchedulingPlan(tuple(plan_from_str(r["plan"])))
        assert not sc(plan).feasible and sc(plan).cost == float.fromhex(r["cost"])
        with pytest.raises(InfeasibleError) as ei:
            provision(plan, g, c, job, mode="stapsratio")
        assert ei.value.gap == 1.0


@pytest.mark.gpu
def test_provisioning_study_matches_reference_rows(tmp_path):
    from paper_2111_10635_b200.studies import provisioning_study
    for it in read_jsonl("study.jsonl.gz"):
        g, c, job = instance(it["instance"])
        rows = provisioning_study(SchedulingPlan(tuple(it["plan"])), g, c, job,
                                  out_dir=tmp_path)
        assert [r.mode for r in rows] == [r["mode"] for r in it["rows"]]
        for got, exp in zip(rows, it["rows"]):
            assert got.feasible == exp["feasible"], (it["plan"], got, exp)
            assert (None if got.cost is None else got.cost.hex()) == exp["cost"]
            assert (None if got.throughput is None else got.throughput.hex()) == exp["throughput"]
            assert (None if got.per_stage_k is None else list(got.per_stage_k)) == exp["k"]
            assert got.ps_cores == exp["ps"]
            assert bool(got.error) == bool(exp["error"])
            if got.mode != "optimal" or "strictly" in exp["error"]:
                assert got.error == exp["error"]
    assert (tmp_path / "provisioning.csv").read_text().startswith("mode,cost,throughput")
