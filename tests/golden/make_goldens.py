"""Generate per-plan golden records by running the REFERENCE scorer (test infrastructure).

Run here (the reference is importable only in the build container):
    python tests/golden/make_goldens.py [--jobs 8]
Outputs under tests/golden/:
  plans_<inst>.jsonl.gz   one record per plan: assignment, cost/gap as float.hex, status,
                          ps, per-stage k, totals order, overflow flag, candidate count
  bf_winners.json         brute-force winners (ls/baselines.py:164-188) for small configs
  kats.json               SPEC.md scalar examples evaluated through the reference
  rng.json                numpy PCG64 / integers / choice vectors (Appendix B of SURVEY.md)
Metadata (python, numpy versions) is stored in meta.json, because the reference's results
depend on CPython>=3.12 builtin sum (Neumaier) and numpy's reduction order.

Status codes (match include/hps.h HPS_ST_*), classified from the reference's exception text:
  0 ok | 1 min_k1 (provisioner.py:96-102) | 2 serial>=tau_hi (:400-412)
  3 quota at tau_hi (:413-427) | 4 floor raise while counting at tau_hi (:164-174 via :414)
  5 no feasible candidate (:473-477) | 6 PS-core quota (:507-512) | 7 defensive evaluate (:481-482)
"""
import argparse
import gzip
import itertools
import json
import multiprocessing as mp
import platform
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import layersched as ls  # noqa: E402
from layersched import provisioner as prov  # noqa: E402

HERE = Path(__file__).resolve().parent
INST = HERE / "instances"

_probe = {"ovf": 0, "ncand": 0}
_orig_best = prov._best_candidate
_orig_golden = prov._golden_minimize


def _best_probe(taus, *a, **k):
    _probe["ncand"] = int(len(taus))
    return _orig_best(taus, *a, **k)


def _golden_probe(*a, **k):
    _probe["ovf"] = 1
    return _orig_golden(*a, **k)


prov._best_candidate = _best_probe
prov._golden_minimize = _golden_probe
_orig_newton = prov._newton_minimize


def _newton_probe(*a, **k):
    _probe["ovf"] = 1
    return _orig_newton(*a, **k)


prov._newton_minimize = _newton_probe


def classify(msg):
    if "serial computation time exceeds the budget" in msg or "serial communication time exceeds the budget" in msg:
        return 1
    if "its serial time" in msg:
        return 2
    if msg.startswith("no count within quota meets the throughput limit: type"):
        return 3
    if "load-balance target" in msg:
        return 4
    if "no count within quota meets the throughput limit strictly" in msg:
        return 5
    if "parameter-server cores" in msg:
        return 6
    if "optimizer produced infeasible plan" in msg:
        return 7
    raise RuntimeError("unclassified infeasibility: " + msg)


def load_instance(name):
    idx = json.loads((INST / "index.json").read_text())[name]
    g = ls.load_model_graph(INST / idx["graph"])
    c = ls.load_catalog(INST / idx["catalog"])
    return g, c, ls.JobParams(idx["throughput_limit"])


_ctx = {}


def _init(name):
    _ctx["inst"] = load_instance(name)


def score_one(assignment):
    g, c, job = _ctx["inst"]
    plan = ls.SchedulingPlan(tuple(int(a) for a in assignment))
    _probe["ovf"] = 0
    _probe["ncand"] = 0
    rec = {"plan": "".join(str(int(a)) if a < 10 else chr(55 + int(a)) for a in assignment)}
    try:
        p = ls.provision(plan, g, c, job)
        rep = ls.evaluate(plan, p, g, c, job)
        rec.update(status=0, cost=rep.monetary_cost.hex(), gap=(0.0).hex(), ps=p.ps_cores,
                   k=list(p.per_stage_k), totals=[[t, n] for t, n in p.per_type_totals.items()],
                   tp=rep.pipeline_throughput.hex(), exec=rep.total_exec_time.hex())
    except ls.InfeasibleError as e:
        pen = ls.scoring.penalty_cost(c, e.gap)
        rec.update(status=classify(str(e)), cost=pen.hex(), gap=e.gap.hex(), ps=0, k=[])
    # scorer view must agree (ls/scoring.py:79-101)
    sc = ls.PlanScorer(g, c, job)(plan)
    assert sc.cost.hex() == rec["cost"], (sc.cost, rec)
    rec["ovf"] = _probe["ovf"]
    rec["ncand"] = _probe["ncand"]
    return rec


def plans_for(name, g, c, rng_seed, n_random):
    T, L = c.num_types, g.num_layers
    if T ** L <= 6561:
        return [tuple(a) for a in itertools.product(range(T), repeat=L)]
    rng = np.random.default_rng(rng_seed)
    return [tuple(int(x) for x in rng.integers(0, T, L)) for _ in range(n_random)]


def write_plans(name, plans, jobs):
    with mp.Pool(jobs, initializer=_init, initargs=(name,)) as pool:
        recs = pool.map(score_one, plans, chunksize=16)
    with gzip.open(HERE / f"plans_{name}.jsonl.gz", "wt") as f:
        for r in recs:
            f.write(json.dumps(r, separators=(",", ":")) + "\n")
    st = np.bincount([r["status"] for r in recs], minlength=8)
    print(name, len(recs), "status", st.tolist(), "ovf", sum(r["ovf"] for r in recs),
          "c1", sum(1 for r in recs if r["ncand"] == 1), flush=True)
    return recs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=8)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    sizes = {"cfg1": 0, "cfg2": 0, "cfg3": 3000, "cfg4": 3000, "cfg5": 600, "quota": 2000,
             "tight16": 2000, "tightmn": 2000, "nce5": 0, "emb2": 1500}
    meta = {"python": platform.python_version(), "numpy": np.__version__,
            "reference": "/root/reference/pkg (layersched 0.1.0)"}
    (HERE / "meta.json").write_text(json.dumps(meta, indent=1) + "\n")
    for name, n in sizes.items():
        if args.only and name not in args.only.split(","):
            continue
        g, c, _ = load_instance(name)
        write_plans(name, plans_for(name, g, c, 12345, n), args.jobs)


if __name__ == "__main__":
    main()
