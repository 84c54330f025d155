"""Parity of the CUDA path (through the C-ABI) with the reference goldens and the oracle.
Bit-exact: cost, gap, status, per-stage counts, PS cores, argmin winners."""
import numpy as np
import pytest

import oracle
from goldens import (PLAN_FILES, expected, inline_instance, instance, plans_array, read_jsonl,
                     staged)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _dev(g, c, job, with_ps=True):
    from paper_2111_10635_b200.instance import DeviceInstance
    return DeviceInstance(g, c, job, with_ps=with_ps)


def _score(inst, plans):
    out = inst.score(torch.from_numpy(np.ascontiguousarray(plans)).cuda())
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}


def _same_bits(a, b):
    return np.array_equal(np.asarray(a, np.float64).view(np.int64), np.asarray(b, np.float64).view(np.int64))


def _check_records(records, out):
    cost, status, gap, ps, ovf = expected(records)
    code = out["status"].astype(np.int64) & 0x7F
    bad = np.flatnonzero(code != status)
    assert bad.size == 0, [(records[i]["plan"], int(code[i]), int(status[i])) for i in bad[:5]]
    bad = np.flatnonzero(out["cost"].view(np.int64) != cost.view(np.int64))
    assert bad.size == 0, [(records[i]["plan"], out["cost"][i], cost[i]) for i in bad[:5]]
    assert _same_bits(out["gap"], gap)
    assert np.array_equal(out["ps"].astype(np.int64), ps)
    assert np.array_equal((out["status"].astype(np.int64) >> 7) & 1, ovf)
    for i, r in enumerate(records):
        if r["status"] == 0:
            S = len(r["k"])
            assert out["num_stages"][i] == S
            assert list(out["k"][i, :S]) == r["k"], r["plan"]


@pytest.mark.parametrize("name", PLAN_FILES)
def test_device_matches_reference_goldens(name):
    records = read_jsonl(f"plans_{name}.jsonl.gz")
    g, c, job = instance(name)
    _check_records(records, _score(_dev(g, c, job), plans_array(records)))


def test_device_overflow_path_matches_reference():
    records = read_jsonl("ovf.jsonl.gz")
    by = {}
    for r in records:
        by.setdefault(r["instance"], []).append(r)
    for name, recs in by.items():
        g, c, job = instance(name)
        _check_records(recs, _score(_dev(g, c, job), plans_array(recs)))


@pytest.mark.parametrize("fname", ["synth.jsonl.gz", "c1.jsonl.gz"])
def test_device_edge_instances_match_reference(fname):
    for it in read_jsonl(fname):
        g, c, job = inline_instance(it)
        recs = [r for r in it["records"] if r["status"] != 255]
        if recs:
            _check_records(recs, _score(_dev(g, c, job), plans_array(recs)))
        inv = [r for r in it["records"] if r["status"] == 255]
        if inv:
            out = _score(_dev(g, c, job), plans_array(inv))
            assert set((out["status"] & 0x7F).tolist()) == {8}


@pytest.mark.parametrize("name,n", [("cfg3", 20000), ("cfg4", 20000), ("cfg5", 4000),
                                    ("tightmn", 20000), ("quota", 20000)])
def test_device_matches_oracle_random_plans(name, n):
    g, c, job = instance(name)
    plans = np.random.default_rng(2024).integers(0, c.num_types, (n, g.num_layers)).astype(np.uint8)
    out = _score(_dev(g, c, job), plans)
    ref = oracle.score_batch(staged(g, c, job), plans)
    assert np.array_equal(out["status"], ref["status"])
    assert _same_bits(out["cost"], ref["cost"])
    assert _same_bits(out["gap"], ref["gap"])
    assert np.array_equal(out["ps"], ref["ps"])
    assert np.array_equal(out["k"], ref["k"])


def test_device_without_ps_matches_oracle():
    g, c, job = instance("cfg4")
    plans = np.random.default_rng(5).integers(0, 2, (3000, 16)).astype(np.uint8)
    out = _score(_dev(g, c, job, with_ps=False), plans)
    ref = oracle.score_batch(staged(g, c, job, with_ps=False), plans)
    assert _same_bits(out["cost"], ref["cost"]) and np.array_equal(out["k"], ref["k"])


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "nce5", "quota"])
def test_enum_argmin_matches_oracle(name):
    g, c, job = instance(name)
    total = c.num_types ** g.num_layers
    inst = _dev(g, c, job)
    key = inst.read_argmin(inst.enum_argmin_async(0, total, True))
    bc, bi, feas = oracle.enum_argmin(staged(g, c, job), 0, total)
    assert (key["cost"], key["rank"], key["feasible"]) == (bc, bi, feas)


def test_enum_argmin_cfg4_full_and_shards():
    g, c, job = instance("cfg4")
    inst = _dev(g, c, job)
    key = inst.read_argmin(inst.enum_argmin_async(0, 2 ** 16, True))
    assert key["rank"] == 4030 and key["cost"] == 0.11630007595486111
    from paper_2111_10635_b200.search import merge_keys, shard_range
    parts = [inst.read_argmin(inst.enum_argmin_async(*shard_range(0, 2 ** 16, r, 8), True))
             for r in range(8)]
    m = merge_keys(parts)
    assert (m["cost"], m["rank"], m["feasible"]) == (key["cost"], key["rank"], key["feasible"])
    from paper_2111_10635_b200.search import enum_shard_async
    for w in (3, 8):   # strided shards, merged like the multi-GPU path
        keys = [inst.read_argmin(enum_shard_async(inst, 0, 2 ** 16, r, w)) for r in range(w)]
        m = merge_keys(keys)
        assert (m["cost"], m["rank"], m["feasible"], m["evaluated"]) == \
            (key["cost"], key["rank"], key["feasible"], 2 ** 16)
    e = inst.read_argmin(inst.enum_argmin_async(5, 5, True))   # empty piece = identity key
    assert e["cost"] == float("inf") and e["evaluated"] == 0 and e["feasible"] == 0


def test_brute_force_dropin_matches_reference_winners():
    import paper_2111_10635_b200 as p
    from paper_2111_10635_b200.search import brute_force
    for name, plan, cost, k, ps in [("cfg1", (0, 0, 1, 1), 0.028293565538194444, (35, 1), 6),
                                    ("cfg2", (0, 0, 0, 0, 0, 1, 1, 1), 0.022149522569444444, (8, 1), 6)]:
        g, c, job = instance(name)
        best = brute_force(g, c, job)
        assert best.plan.assignment == plan and best.cost == cost
        assert best.provisioning.per_stage_k == k and best.provisioning.ps_cores == ps
        assert best.evaluations == c.num_types ** g.num_layers


def test_random_argmin_matches_oracle_stream():
    from paper_2111_10635_b200.instance import pcg_from_generator
    from paper_2111_10635_b200.search import decode_packed
    g, c, job = instance("cfg5")
    inst = _dev(g, c, job)
    n = 3000
    pcg = pcg_from_generator(np.random.default_rng(0))
    plans_dev = inst.random_plans(pcg, 0, n).cpu().numpy()
    rng = np.random.default_rng(0)
    ref_plans = np.stack([rng.integers(0, 4, 64) for _ in range(n)]).astype(np.uint8)
    assert np.array_equal(plans_dev, ref_plans)
    # shifted start (plan 1000) = the same stream
    assert np.array_equal(inst.random_plans(pcg, 1000, 50).cpu().numpy(), ref_plans[1000:1050])
    key = inst.read_argmin(inst.random_argmin_async(pcg, 0, n))
    ref = oracle.score_batch(staged(g, c, job), ref_plans)
    order = sorted(range(n), key=lambda i: (ref["cost"][i], tuple(ref_plans[i])))
    assert key["cost"] == ref["cost"][order[0]]
    assert decode_packed(key["rank"], 4, 64) == tuple(int(x) for x in ref_plans[order[0]])


def test_plans_argmin_non_power_of_two():
    g, c, job = instance("cfg3")
    inst = _dev(g, c, job)
    plans = np.random.default_rng(9).integers(0, 3, (5000, 16)).astype(np.uint8)
    key = inst.read_argmin(inst.plans_argmin_async(torch.from_numpy(plans).cuda(), False))
    ref = oracle.score_batch(staged(g, c, job), plans)
    i = min(range(len(plans)), key=lambda i: (ref["cost"][i], tuple(plans[i])))
    from paper_2111_10635_b200.search import decode_packed
    assert key["cost"] == ref["cost"][i] and decode_packed(key["rank"], 3, 16) == tuple(int(x) for x in plans[i])


def test_scorer_dropin_reports_match_goldens():
    from paper_2111_10635_b200.scoring import PlanScorer, evaluate, provision
    from paper_2111_10635_b200.model import SchedulingPlan
    records = [r for r in read_jsonl("plans_cfg4.jsonl.gz") if r["status"] == 0][:200]
    g, c, job = instance("cfg4")
    sc = PlanScorer(g, c, job)
    from goldens import plan_from_str
    scored = sc.score_many([SchedulingPlan(tuple(plan_from_str(r["plan"]))) for r in records])
    for r, s in zip(records, scored):
        assert s.cost.hex() == r["cost"] and list(s.provisioning.per_stage_k) == r["k"]
        assert [[t, n] for t, n in s.provisioning.per_type_totals.items()] == r["totals"]
        assert s.report.pipeline_throughput.hex() == r["tp"]
        assert s.report.total_exec_time.hex() == r["exec"]
        assert s.report.monetary_cost.hex() == r["cost"]
    p0 = SchedulingPlan(tuple(plan_from_str(records[0]["plan"])))
    prov = provision(p0, g, c, job)
    rep = evaluate(p0, prov, g, c, job)
    assert rep.monetary_cost.hex() == records[0]["cost"] and rep.feasible


@pytest.mark.parametrize("name,n", [("cfg3", 30000), ("cfg5", 3000), ("quota", 20000), ("tightmn", 20000)])
def test_fast_path_equals_literal_path(name, n, monkeypatch):
    """The threshold-table sweep (default) and the literal division path agree bit for bit."""
    g, c, job = instance(name)
    plans = np.random.default_rng(77).integers(0, c.num_types, (n, g.num_layers)).astype(np.uint8)
    fast = _score(_dev(g, c, job), plans)
    monkeypatch.setenv("HPS_FORCE_LITERAL", "1")
    lit = _score(_dev(g, c, job), plans)
    for k in ("status", "ps", "k", "num_stages"):
        assert np.array_equal(fast[k], lit[k]), k
    assert _same_bits(fast["cost"], lit["cost"]) and _same_bits(fast["gap"], lit["gap"])
