"""Full-sweep goldens: winner, feasible count, per-status counts and the order-independent digest
of EVERY plan's outputs, for each exhaustive configuration (test infrastructure).

    python tests/golden/make_sweep_digests.py [--threads 8] [--only cfg3]

The sweep runs on the C oracle (oracle/hps_oracle.c, itself pinned bit-for-bit to the reference
by tests/test_oracle_golden.py): the reference's own brute_force refuses T^L > 2^24
(ls/baselines.py:27,73-78), and scoring 3^16 plans with the Python reference would take ~33 h on
one core. The reference is still consulted here, for every winner: its PlanScorer
(ls/scoring.py:79-101) must return the same cost for the winning plan, and for the configs it
accepts (T^L <= 2^16 here) its brute_force (ls/baselines.py:63-87) must return the same plan.
Output: tests/golden/sweep_digests.json (read by tests/test_gpu_sweep.py).
"""
import argparse
import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

import layersched as ls  # noqa: E402

import oracle  # noqa: E402
from goldens import instance, staged  # noqa: E402
from make_goldens import load_instance  # noqa: E402

OUT = HERE / "sweep_digests.json"
CONFIGS = ["cfg1", "cfg2", "nce5", "quota", "cfg4", "cfg3"]


def decode(idx, T, L):
    d = []
    for _ in range(L):
        d.append(idx % T)
        idx //= T
    return tuple(reversed(d))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=8)
    ap.add_argument("--only", nargs="*")
    a = ap.parse_args()
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    for name in a.only or CONFIGS:
        g, c, job = instance(name)
        T, L = c.num_types, g.num_layers
        total = T ** L
        t0 = time.time()
        r = oracle.enum_digest(staged(g, c, job), 0, total, a.threads)
        dt = time.time() - t0
        rg, rc, rj = load_instance(name)
        plan = ls.SchedulingPlan(decode(r["best_index"], T, L))
        ref_cost = ls.PlanScorer(rg, rc, rj)(plan).cost
        assert ref_cost == r["best_cost"], (name, ref_cost, r)
        if total <= 1 << 16:
            bf = ls.brute_force(rg, rc, rj)
            assert tuple(bf.plan.assignment) == plan.assignment and bf.cost == r["best_cost"], name
        data[name] = {"plans": total, "best_index": r["best_index"], "best_plan": list(plan.assignment),
                      "best_cost": r["best_cost"].hex(), "feasible": r["feasible"],
                      "digest": str(r["digest"]), "overflow": r["overflow"],
                      "by_status": {str(k): v for k, v in r["by_status"].items()},
                      "oracle_seconds": round(dt, 1), "threads": a.threads}
        print(name, data[name], flush=True)
        OUT.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
