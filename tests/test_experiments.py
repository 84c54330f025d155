"""Experiment harness (ls/experiments.py) on the device drop-ins: run_method for every method
and the scaling study vs the reference's own outputs (tests/golden/make_experiment_goldens.py),
plus the CSV / plan-file round trips."""
import gzip
import json

import pytest

from goldens import GOLDEN, instance
from paper_2111_10635_b200 import experiments as ex
from paper_2111_10635_b200.errors import ConfigError
from paper_2111_10635_b200.model import JobParams, ProvisioningPlan, ScoredPlan, SchedulingPlan

with gzip.open(GOLDEN / "experiments.json.gz", "rt") as _f:
    GOLD = json.load(_f)
MCFG = {"genetic": {"population": 12, "generations": 5}, "random": {"budget": 64},
        "rl-lstm": {"rounds": 6, "plans_per_round": 32},
        "rl-rnn": {"rounds": 6, "plans_per_round": 32}}


def test_comparison_csv_round_trips_exactly(tmp_path):
    rows = [ex.ComparisonRow("bf", 0, "m", (0, 1, 1), 0.1 + 0.2, 300.00000000000006, 5e4 / 3,
                             1.0 / 3, 0.125, True),
            ex.ComparisonRow("rl-lstm", 2, "m", None, None, None, None, None, 1e-3, False,
                             "no feasible provisioning")]
    p = tmp_path / "comparison.csv"
    ex.write_comparison_csv(p, rows, 1000.0)
    back, norm = ex.read_comparison_csv(p)
    assert back == rows and norm == 1000.0
    files = ex.emit_plot_data(rows, tmp_path)
    assert [f.name for f in files] == ["cost_by_method.csv", "throughput_by_method.csv",
                                       "cost_by_model.csv"]
    assert files[0].read_text().splitlines()[1] == "bf,0,0.30000000000000004,300.00000000000006"


def test_plan_file_round_trip(tmp_path):
    g, c, job = instance("cfg1")
    s = ScoredPlan(SchedulingPlan((0, 0, 1, 1)), ProvisioningPlan((35, 1), 6, {0: 41, 1: 1}),
                   0.028293565538194444)
    ex.write_plan_file(tmp_path / "p.json", g, s)
    plan, prov = ex.read_plan_file(tmp_path / "p.json")
    assert plan == s.plan and prov == s.provisioning
    with pytest.raises(ConfigError):
        ex.read_plan_file(tmp_path / "missing.json")


def test_experiment_config_validation(tmp_path):
    with pytest.raises(ConfigError):
        ex.ExperimentConfig("m", "c", 1.0, ())
    with pytest.raises(ConfigError):
        ex.ExperimentConfig("m", "c", 1.0, ("nope",))
    (tmp_path / "e.json").write_text(json.dumps({"model": "m", "catalog": "c",
                                                 "throughput_limit": 5, "methods": ["bf"]}))
    cfg = ex.load_experiment_config(tmp_path / "e.json")
    assert cfg.methods == ("bf",) and cfg.seeds == (0,) and cfg.cost_normalization == 1000.0


@pytest.mark.gpu
def test_run_method_matches_reference_for_every_method():
    cache = {}
    for rec in GOLD["run_method"]:
        if rec["instance"] not in cache:
            cache[rec["instance"]] = instance(rec["instance"])
        g, c, job = cache[rec["instance"]]
        if "error" in rec:
            with pytest.raises(Exception) as ei:
                ex.run_method(rec["method"], g, c, job, rec["seed"], MCFG)
            assert str(ei.value) == rec["error"]
            continue
        s = ex.run_method(rec["method"], g, c, job, rec["seed"], MCFG)
        assert (list(s.plan.assignment), s.cost.hex(), s.feasible, s.evaluations) == \
            (rec["plan"], rec["cost"], rec["feasible"], rec["evaluations"]), rec


@pytest.mark.gpu
def test_scaling_study_matches_reference_costs(tmp_path):
    from paper_2111_10635_b200.policy import TrainerConfig
    g, c, _ = instance("cfg4")   # ctrdnn16 + catalog_default, like the reference's bundled pair
    rows = ex.scaling_study((2, 3, 4), (2, 3), g, c, JobParams(5e4),
                            TrainerConfig(rounds=5, plans_per_round=8), bf_time_cap_s=600,
                            out_dir=tmp_path)
    got = [{"layers": r.layers, "types": r.types, "enumerations": r.enumerations,
            "bf_cost": None if r.bf_cost is None else r.bf_cost.hex(),
            "rl_cost": None if r.rl_cost is None else r.rl_cost.hex()} for r in rows]
    assert got == GOLD["scaling"]
    assert all(not r.bf_estimated for r in rows)
    assert (tmp_path / "scaling.csv").read_text().startswith(",".join(ex.SCALING_COLUMNS))


@pytest.mark.gpu
def test_timed_enumeration_cap_extrapolates():
    g, c, job = instance("cfg3")
    total, est, estimated, best = ex.timed_enumeration(g, c, job, 0.0, chunk=1 << 20)
    assert total == 3 ** 16 and estimated and best is None and est > 0
    g, c, job = instance("cfg2")
    total, wall, estimated, best = ex.timed_enumeration(g, c, job, 60.0)
    assert (total, estimated, best) == (6561, False, 0.022149522569444444)


@pytest.mark.gpu
def test_run_experiment_writes_rows_csvs_and_plans(tmp_path):
    g, c, job = instance("cfg2")
    cfg = ex.ExperimentConfig("cfg2", "cat", job.throughput_limit, ("bf", "greedy", "cpu"),
                              seeds=(0,), out_dir=str(tmp_path))
    rows = ex.run_experiment(cfg, g, c)
    assert [r.method for r in rows] == ["bf", "greedy", "cpu"]
    assert rows[0].cost == 0.022149522569444444 and rows[0].feasible
    back, _ = ex.read_comparison_csv(tmp_path / "comparison.csv")
    assert [r.cost for r in back] == [r.cost for r in rows]
    assert (tmp_path / "plan_bf_s0.json").exists()
