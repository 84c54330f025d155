"""Golden results of the REFERENCE's greedy / genetic / heuristic / homogeneous / dedup random
searchers (ls/baselines.py:90-282) on the fixtures (test infrastructure; run here only)."""
import gzip
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent))
import layersched as ls  # noqa: E402
from layersched import baselines as bl  # noqa: E402
import make_goldens as mg  # noqa: E402

HERE = Path(__file__).resolve().parent


def sp(s):
    return {"plan": list(s.plan.assignment), "cost": s.cost.hex(), "evaluations": s.evaluations,
            "feasible": s.feasible}


def main():
    out = []
    for name in ("cfg1", "cfg2", "cfg4", "quota", "nce5", "tightmn"):
        g, c, job = mg.load_instance(name)
        rec = {"instance": name, "greedy": sp(bl.greedy(g, c, job))}
        gens = []
        for seed, pop, gen in ((0, 16, 8), (1, 8, 5), (3, 64, 12)):
            cfg = bl.GeneticConfig(population=pop, generations=gen, seed=seed)
            gens.append({"seed": seed, "population": pop, "generations": gen,
                         "result": sp(bl.genetic(g, c, job, cfg))})
        cfg = bl.GeneticConfig(population=12, generations=6, seed=5, crossover_rate=0.3,
                               mutation_rate=0.4, tournament_size=2)
        seeds = [bl.homogeneous(g, c, t) for t in range(c.num_types)]
        gens.append({"seed": 5, "population": 12, "generations": 6, "crossover_rate": 0.3,
                     "mutation_rate": 0.4, "tournament_size": 2, "seed_plans": "homogeneous",
                     "result": sp(bl.genetic(g, c, job, cfg, seed_plans=seeds))})
        rec["genetic"] = gens
        try:
            rec["heuristic"] = [list(bl.heuristic_first_layer(g, c, inv).assignment) for inv in (False, True)]
        except ls.SchedulerError as e:
            rec["heuristic"] = str(e)
        rec["random_dedup"] = [dict(budget=b, seed=s, result=sp(bl.random_search(g, c, job, b, s, dedup=True)))
                               for b, s in ((50, 0), (300, 7))]
        out.append(rec)
        print(name, rec["greedy"]["cost"], [x["result"]["cost"] for x in gens])
    with gzip.open(HERE / "search.jsonl.gz", "wt") as f:
        for it in out:
            f.write(json.dumps(it, separators=(",", ":")) + "\n")


if __name__ == "__main__":
    main()
