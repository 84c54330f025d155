"""RL golden traces from the REFERENCE trainer (test infrastructure; run here only).

For cfg1 (CTRDNN-4, T=2, G=64, R=200, seeds 0-2) and cfg4 (CTRDNN16, T=2, G=4096, first 12
rounds, seed 0; `--cfg4-full`: all 200 rounds into rl_traces_cfg4_200.json.gz), record per round: RoundStats (mean_cost, best_cost, baseline, entropy as
float.hex), a digest of the sampled plans (sha1 of the G x L action bytes), the number of
infeasible plans, and the final parameters' checksum/norm; plus init parameters checksum.
ls/policy/training.py:164-274 is run unmodified; sampling is observed by wrapping
ls/policy/network.sample_actions (the function train() calls, training.py:206).
"""
import gzip
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import layersched as ls  # noqa: E402
from layersched.policy import training as tr  # noqa: E402

HERE = Path(__file__).resolve().parent


def load(name):
    idx = json.loads((HERE / "instances" / "index.json").read_text())[name]
    g = ls.load_model_graph(HERE / "instances" / idx["graph"])
    c = ls.load_catalog(HERE / "instances" / idx["catalog"])
    return g, c, ls.JobParams(idx["throughput_limit"])


def run(name, seed, rounds, G):
    g, c, job = load(name)
    cfg = tr.TrainerConfig(rounds=rounds, plans_per_round=G, seed=seed)
    params0, norm = tr.init_policy(g, c, cfg)
    log = {"actions": []}
    orig = tr.sample_actions

    def spy(probs, rng):
        a, lp = orig(probs, rng)
        log["actions"].append(np.asarray(a, dtype=np.uint8).copy())
        return a, lp

    tr.sample_actions = spy
    try:
        res = tr.train(g, c, params0, cfg, job)
    finally:
        tr.sample_actions = orig
    acts = np.stack(log["actions"]).reshape(rounds, G, g.num_layers)
    rounds_out = []
    for r, st in enumerate(res.history):
        rounds_out.append({
            "round": st.round, "mean_cost": st.mean_cost.hex(), "best_cost": st.best_cost.hex(),
            "baseline": st.baseline.hex(), "entropy": st.entropy.hex(),
            "plans_sha1": hashlib.sha1(acts[r].tobytes()).hexdigest()})
    flat0 = params0.flat()
    flat = res.params.flat()
    return {"instance": name, "seed": seed, "rounds": rounds, "plans_per_round": G,
            "init_params_sha1": hashlib.sha1(flat0.tobytes()).hexdigest(),
            "init_params_sum": float(flat0.sum()).hex(),
            "final_params_norm": float(np.linalg.norm(flat)).hex(),
            "final_params_sum": float(flat.sum()).hex(),
            "best_plan": list(res.best.plan.assignment), "best_cost": res.best.cost.hex(),
            "first_round_actions": acts[0].tolist() if G <= 64 else acts[0, :64].tolist(),
            "history": rounds_out}


def main():
    if "--cfg4-full" in sys.argv:   # all 200 rounds of BASELINE cfg4 (~7 min on one core)
        tr4 = run("cfg4", 0, 200, 4096)
        print("cfg4 best", tr4["best_plan"], float.fromhex(tr4["best_cost"]), flush=True)
        with gzip.open(HERE / "rl_traces_cfg4_200.json.gz", "wt") as f:
            json.dump(tr4, f)
        return
    out = []
    for seed in (0, 1, 2):
        out.append(run("cfg1", seed, 200, 64))
        print("cfg1 seed", seed, "best", out[-1]["best_plan"], float.fromhex(out[-1]["best_cost"]), flush=True)
    out.append(run("cfg4", 0, 12, 4096))
    print("cfg4 best", out[-1]["best_plan"], float.fromhex(out[-1]["best_cost"]), flush=True)
    with gzip.open(HERE / "rl_traces.json.gz", "wt") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
