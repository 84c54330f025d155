"""Golden outputs of the REFERENCE's experiment harness (ls/experiments.py): run_method for
every method and the scaling study's brute-force / RL costs (test infrastructure; run here)."""
import gzip
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent))
import layersched as ls  # noqa: E402
from layersched import experiments as ex  # noqa: E402
from layersched.policy import TrainerConfig  # noqa: E402
import make_goldens as mg  # noqa: E402

HERE = Path(__file__).resolve().parent
MCFG = {"genetic": {"population": 12, "generations": 5},
        "random": {"budget": 64},
        "rl-lstm": {"rounds": 6, "plans_per_round": 32},
        "rl-rnn": {"rounds": 6, "plans_per_round": 32}}


def main():
    out = {"run_method": [], "scaling": []}
    for name in ("cfg1", "cfg2", "cfg4"):
        g, c, job = mg.load_instance(name)
        for m in ex.METHODS:
            if m == "bf" and c.num_types ** g.num_layers > 70000:
                continue
            for seed in (0, 1):
                try:
                    s = ex.run_method(m, g, c, job, seed, MCFG)
                    rec = {"plan": list(s.plan.assignment), "cost": s.cost.hex(),
                           "feasible": s.feasible, "evaluations": s.evaluations}
                except ls.SchedulerError as e:
                    rec = {"error": str(e)}
                out["run_method"].append({"instance": name, "method": m, "seed": seed, **rec})
    g, c, job = mg.load_instance("cfg1")
    rows = ex.scaling_study((2, 3, 4), (2, 3), ls.load_bundled_graph("ctrdnn16"),
                            ls.load_bundled_catalog(), ls.JobParams(5e4),
                            TrainerConfig(rounds=5, plans_per_round=8), bf_time_cap_s=600)
    out["scaling"] = [{"layers": r.layers, "types": r.types, "enumerations": r.enumerations,
                       "bf_cost": None if r.bf_cost is None else r.bf_cost.hex(),
                       "rl_cost": None if r.rl_cost is None else r.rl_cost.hex()} for r in rows]
    with gzip.open(HERE / "experiments.json.gz", "wt") as f:
        json.dump(out, f)
    print(len(out["run_method"]), "run_method records;", out["scaling"])


if __name__ == "__main__":
    main()
