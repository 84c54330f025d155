"""cfg4 RL training timed per round (device events), graph-replayed and eager; for ncu launch
lists use --rounds 3 (not a bench)."""
import argparse
import os
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instance", default="cfg4")
    ap.add_argument("--rounds", type=int, default=200)
    ap.add_argument("--plans", type=int, default=4096)
    ap.add_argument("--modes", default="graph,eager")
    a = ap.parse_args()
    import torch
    from paper_2111_10635_b200 import load_fixture, policy
    from paper_2111_10635_b200.model import JobParams
    g, c, limit = load_fixture(a.instance)
    job = JobParams(limit)
    cfg = policy.TrainerConfig(rounds=a.rounds, plans_per_round=a.plans, seed=0)
    p0, _ = policy.init_policy(g, c, cfg)
    res = {}
    for mode in a.modes.split(","):
        os.environ["HPS_RL_GRAPH"] = "1" if mode == "graph" else "0"
        policy.train(g, c, p0, policy.TrainerConfig(rounds=2, plans_per_round=a.plans, seed=0), job, shard=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = policy.train(g, c, p0, cfg, job, shard=False)
        wall = time.perf_counter() - t0
        w = r.round_wall_s
        per = [b - a_ for a_, b in zip([0.0] + w[:-1], w)]
        res[mode] = r
        print(f"{mode}: wall {wall:.4f} s, device {w[-1]:.4f} s, round median {1e3 * statistics.median(per):.3f} ms, "
              f"first {1e3 * per[0]:.3f} ms, best {r.best.cost!r}", flush=True)
    if len(res) == 2:
        ra, rb = res.values()
        same = all(x.best_cost == y.best_cost and x.baseline == y.baseline and x.mean_cost == y.mean_cost
                   for x, y in zip(ra.history, rb.history))
        print("graph == eager history:", same, " params equal:",
              bool((ra.params.flat() == rb.params.flat()).all()))


if __name__ == "__main__":
    main()
