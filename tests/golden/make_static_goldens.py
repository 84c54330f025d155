"""Golden records for the static provisioning modes (ls/provisioner.py:516-561), from the
REFERENCE's PlanScorer(mode='staratio' | 'stapsratio') (test infrastructure; run here only)."""
import gzip
import itertools
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent))
import layersched as ls  # noqa: E402
import make_goldens as mg  # noqa: E402
from make_edge_goldens import rand_instance  # noqa: E402
from layersched.fileio import graph_to_dict, catalog_to_dict  # noqa: E402

HERE = Path(__file__).resolve().parent


def PS(a):
    return "".join(str(int(x)) if x < 10 else chr(55 + int(x)) for x in a)


def rec(g, c, job, a, mode):
    plan = ls.SchedulingPlan(tuple(a))
    try:
        sc = ls.PlanScorer(g, c, job, mode=mode)(plan)
    except ls.InvariantError:
        return {"plan": PS(a), "status": 255}
    out = {"plan": PS(a), "cost": sc.cost.hex()}
    if sc.feasible:
        p = sc.provisioning
        out.update(status=0, k=list(p.per_stage_k), ps=p.ps_cores,
                   totals=[[t, n] for t, n in p.per_type_totals.items()])
    else:
        out.update(status=10)
    return out


def main():
    items = []
    for name in ("cfg1", "cfg2", "cfg4", "quota", "nce5"):
        g, c, job = mg.load_instance(name)
        T, L = c.num_types, g.num_layers
        if T ** L <= 6561:
            plans = list(itertools.product(range(T), repeat=L))
        else:
            rng = np.random.default_rng(7)
            plans = [tuple(int(x) for x in rng.integers(0, T, L)) for _ in range(1500)]
        for mode in ("staratio", "stapsratio"):
            items.append({"instance": name, "mode": mode, "records": [rec(g, c, job, a, mode) for a in plans]})
    rng = np.random.default_rng(4242)
    for i in range(120):
        g, c, limit = rand_instance(rng)
        job = ls.JobParams(limit)
        plans = list(itertools.product(range(c.num_types), repeat=g.num_layers))[:300]
        for mode in ("staratio", "stapsratio"):
            items.append({"graph": graph_to_dict(g), "catalog": catalog_to_dict(c), "throughput_limit": limit,
                          "mode": mode, "records": [rec(g, c, job, a, mode) for a in plans]})
    with gzip.open(HERE / "static.jsonl.gz", "wt") as f:
        for it in items:
            f.write(json.dumps(it, separators=(",", ":")) + "\n")
    st = [r["status"] for it in items for r in it["records"]]
    print("records", len(st), "feasible", st.count(0), "infeasible", st.count(10), "invariant", st.count(255))


if __name__ == "__main__":
    main()
