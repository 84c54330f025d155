"""greedy / genetic / heuristic / homogeneous / dedup random search vs the reference's own
results (tests/golden/make_search_goldens.py, ls/baselines.py:90-282)."""
import pytest

from goldens import instance, read_jsonl
from paper_2111_10635_b200 import search
from paper_2111_10635_b200.errors import InvariantError, PlanValidationError

ITEMS = read_jsonl("search.jsonl.gz")


def _same(res, exp):
    assert list(res.plan.assignment) == exp["plan"]
    assert res.cost.hex() == exp["cost"]
    assert res.evaluations == exp["evaluations"]
    assert res.feasible == exp["feasible"]


@pytest.mark.parametrize("it", ITEMS, ids=[it["instance"] for it in ITEMS])
def test_heuristic_and_homogeneous_match_reference(it):
    g, c, job = instance(it["instance"])
    if isinstance(it["heuristic"], str):
        with pytest.raises(Exception) as ei:
            search.heuristic_first_layer(g, c)
        assert str(ei.value) == it["heuristic"]
    else:
        got = [list(search.heuristic_first_layer(g, c, inv).assignment) for inv in (False, True)]
        assert got == it["heuristic"]
    assert search.homogeneous(g, c, 0).assignment == (0,) * g.num_layers
    with pytest.raises(PlanValidationError):
        search.homogeneous(g, c, c.num_types)


def test_genetic_config_validation():
    with pytest.raises(InvariantError):
        search.GeneticConfig(population=1)
    with pytest.raises(InvariantError):
        search.GeneticConfig(mutation_rate=1.5)


@pytest.mark.gpu
@pytest.mark.parametrize("it", ITEMS, ids=[it["instance"] for it in ITEMS])
def test_device_searchers_match_reference(it):
    g, c, job = instance(it["instance"])
    _same(search.greedy(g, c, job), it["greedy"])
    for gcfg in it["genetic"]:
        cfg = search.GeneticConfig(population=gcfg["population"], generations=gcfg["generations"],
                                   seed=gcfg["seed"],
                                   crossover_rate=gcfg.get("crossover_rate", 0.8),
                                   mutation_rate=gcfg.get("mutation_rate"),
                                   tournament_size=gcfg.get("tournament_size", 3))
        seeds = ([search.homogeneous(g, c, t) for t in range(c.num_types)]
                 if gcfg.get("seed_plans") else ())
        _same(search.genetic(g, c, job, cfg, seed_plans=seeds), gcfg["result"])
    for r in it["random_dedup"]:
        _same(search.random_search(g, c, job, r["budget"], r["seed"], dedup=True), r["result"])
