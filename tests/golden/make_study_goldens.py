"""Golden rows of the REFERENCE's provisioning_study (ls/experiments.py:637-703) for a few
plans per instance, including the error text (test infrastructure; run here only)."""
import gzip
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent))
import layersched as ls  # noqa: E402
from layersched.experiments import provisioning_study  # noqa: E402
import make_goldens as mg  # noqa: E402

HERE = Path(__file__).resolve().parent


def main():
    out = []
    for name, n in (("cfg1", 16), ("cfg2", 60), ("cfg4", 40), ("quota", 40), ("nce5", 40)):
        g, c, job = mg.load_instance(name)
        rng = np.random.default_rng(11)
        for _ in range(n):
            a = tuple(int(x) for x in rng.integers(0, c.num_types, g.num_layers))
            rows = provisioning_study(ls.SchedulingPlan(a), g, c, job)
            out.append({"instance": name, "plan": list(a), "rows": [
                {"mode": r.mode, "cost": None if r.cost is None else r.cost.hex(),
                 "throughput": None if r.throughput is None else r.throughput.hex(),
                 "k": None if r.per_stage_k is None else list(r.per_stage_k),
                 "ps": r.ps_cores, "feasible": r.feasible, "error": r.error} for r in rows]})
    with gzip.open(HERE / "study.jsonl.gz", "wt") as f:
        for it in out:
            f.write(json.dumps(it, separators=(",", ":")) + "\n")
    rows = [r for it in out for r in it["rows"]]
    print(len(out), "plans", sum(r["feasible"] for r in rows), "feasible rows",
          sorted({r["error"].split(":")[0][:50] for r in rows if r["error"]}))


if __name__ == "__main__":
    main()
