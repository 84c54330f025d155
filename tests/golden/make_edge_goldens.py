"""Edge-case golden records from the REFERENCE (test infrastructure; run here only).

  synth.jsonl.gz   random small instances (L<=7, T<=4) with zero profiles, alpha/beta in
                   {0,1}, tiny quotas, CPU-less catalogs, extreme limits -- every plan of each
                   instance is scored, so every infeasibility branch of
                   ls/provisioner.py:80-513 and ls/scoring.py:79-101 is exercised.
  c1.jsonl.gz      constructed single-candidate cases (tau_lo == tau_hi), the only branch where
                   _best_candidate's per_second uses numpy's pairwise sum (provisioner.py:306).
  ovf.jsonl.gz     plans taking the >4096-breakpoint path (Newton/golden/subsample,
                   provisioner.py:456-470), mined from large random samples of bundled instances.
Each record carries its instance inline (graph/catalog dicts + limit) or an instance name.
"""
import gzip
import itertools
import json
import math
import multiprocessing as mp
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent))
import layersched as ls  # noqa: E402
from layersched.fileio import graph_to_dict, catalog_to_dict  # noqa: E402
import make_goldens as mg  # noqa: E402

HERE = Path(__file__).resolve().parent


def rand_instance(rng, L=None, T=None):
    L = int(rng.integers(1, 8)) if L is None else L
    T = int(rng.integers(1, 5)) if T is None else T
    while T ** L > 2500:
        L -= 1
    types = []
    ncpu = 0
    for t in range(T):
        is_cpu = bool(rng.random() < 0.4) or (t == 0 and rng.random() < 0.9)
        ncpu += is_cpu
        quota = int(rng.choice([1, 2, 3, 5, 8, 13, 40, 200, 1000, 10000]))
        price = float(rng.choice([0.04, 2.42, 0.5, 1.0, 3.0])) * (1.0 + 0.1 * int(rng.integers(0, 3)))
        types.append(ls.ResourceType(t, f"t{t}", price, "u", quota, is_cpu))
    cat = ls.ResourceCatalog(tuple(types))

    def val(scale):
        r = rng.random()
        if r < 0.12:
            return 0.0
        return float(rng.uniform(0.001, 1.0) * scale)

    def frac():
        r = rng.random()
        if r < 0.1:
            return 0.0
        if r < 0.2:
            return 1.0
        return float(rng.uniform(0.5, 0.999))

    layers = []
    for l in range(L):
        layers.append(ls.LayerSpec(
            index=l, layer_kind="full-connection", input_size=1e6, weight_size=1e6,
            per_type_oct={t: val(3.0) for t in range(T)},
            per_type_odt={t: val(1.0) for t in range(T)},
            per_type_alpha={t: frac() for t in range(T)},
            per_type_beta={t: frac() for t in range(T)}))
    bo = int(rng.choice([1, 8, 32, 48]))
    batch = int(rng.choice([64, 512, 1000]))
    g = ls.ModelGraph("synth", tuple(layers), total_samples=int(rng.choice([4000000, 123457])),
                      epochs=int(rng.choice([1, 3])), batch_size=batch, profile_batch_size=bo)
    r = rng.random()
    if r < 0.25:  # tiny limits reach min_k1 (provisioner.py:96) and the k1_floor>1 branch (:396)
        limit = float(10 ** rng.uniform(-3.0, 0.5))
    else:  # limits near the instance's own scale keep most plans feasible-ish
        mean_oct = float(np.mean([v for l in layers for v in l.per_type_oct.values()]) + 1e-3)
        limit = batch * bo / (mean_oct * float(rng.uniform(0.02, 3.0)))
    return g, cat, limit




def score_with(g, c, limit, assignment):
    mg._ctx["inst"] = (g, c, ls.JobParams(limit))
    try:
        return mg.score_one(assignment)
    except ls.InvariantError as e:  # CPU-less catalog with accelerator units (domain.py:163-167)
        return {"plan": "".join(map(str, assignment)), "status": 255, "error": "InvariantError"}


def synth_worker(seed):
    rng = np.random.default_rng([seed, 77])
    g, c, limit = rand_instance(rng)
    recs = []
    for a in itertools.product(range(c.num_types), repeat=g.num_layers):
        recs.append(score_with(g, c, limit, a))
    return {"graph": graph_to_dict(g), "catalog": catalog_to_dict(c), "throughput_limit": limit,
            "records": recs}


def c1_worker(seed):
    """Tune the limit so tau_hi = batch/limit sits one ulp above the serial floor."""
    rng = np.random.default_rng([seed, 91])
    out = []
    for it in range(40):
        if it % 2:  # many alternating stages so the pairwise branch (S>=8) is reached
            g, c, limit = rand_instance(rng, L=int(rng.integers(8, 14)), T=2)
            a = tuple(i % 2 for i in range(g.num_layers))
        else:
            g, c, limit = rand_instance(rng)
            a = tuple(int(x) for x in rng.integers(0, c.num_types, g.num_layers))
        plan = ls.SchedulingPlan(a)
        stages = ls.build_stages(plan, g)
        bo = g.profile_batch_size
        serial = ls.provisioner._serial_floor(stages, bo)
        if not serial > 0:
            continue
        target = math.nextafter(serial, math.inf)
        lim = g.batch_size / target
        for _ in range(8):
            if g.batch_size / lim == target:
                break
            lim = math.nextafter(lim, math.inf if g.batch_size / lim > target else 0.0)
        if g.batch_size / lim != target:
            continue
        r = score_with(g, c, lim, a)
        if r.get("ncand") == 1 or r["status"] in (4, 5, 7):
            out.append({"graph": graph_to_dict(g), "catalog": catalog_to_dict(c),
                        "throughput_limit": lim, "records": [r]})
    return out


def ovf_worker(args):
    name, seed, n = args
    g, c, job = mg.load_instance(name)
    rng = np.random.default_rng([seed, 5])
    found = []
    for _ in range(n):
        a = tuple(int(x) for x in rng.integers(0, c.num_types, g.num_layers))
        mg._ctx["inst"] = (g, c, job)
        r = mg.score_one(a)
        if r["ovf"]:
            r["instance"] = name
            found.append(r)
    return found


def dump(name, items):
    with gzip.open(HERE / name, "wt") as f:
        for it in items:
            f.write(json.dumps(it, separators=(",", ":")) + "\n")


def main():
    with mp.Pool(8) as pool:
        synth = pool.map(synth_worker, range(600), chunksize=4)
        dump("synth.jsonl.gz", synth)
        st = np.bincount([r["status"] for s in synth for r in s["records"] if r["status"] < 255],
                         minlength=8)
        print("synth instances", len(synth), "plans", sum(len(s["records"]) for s in synth),
              "status", st.tolist(), "ovf", sum(r.get("ovf", 0) for s in synth for r in s["records"]),
              "c1", sum(1 for s in synth for r in s["records"] if r.get("ncand") == 1),
              "invariant", sum(1 for s in synth for r in s["records"] if r["status"] == 255))
        c1 = [x for lst in pool.map(c1_worker, range(400)) for x in lst]
        dump("c1.jsonl.gz", c1)
        print("c1 cases", len(c1), "ncand==1:", sum(1 for x in c1 if x["records"][0].get("ncand") == 1),
              "with S>=8:", sum(1 for x in c1 if len(x["records"][0].get("k", [])) >= 8
                                and x["records"][0].get("ncand") == 1),
              "status", np.bincount([x["records"][0]["status"] for x in c1 if x["records"][0]["status"] < 255], minlength=8).tolist())
        jobs = [(n, s, 1500) for n in ("tightmn", "cfg5", "cfg4", "tight16") for s in range(8)]
        ovf = [x for lst in pool.map(ovf_worker, jobs) for x in lst]
        dump("ovf.jsonl.gz", ovf)
        print("ovf plans", len(ovf), {n: sum(1 for r in ovf if r["instance"] == n)
                                     for n in ("tightmn", "cfg5", "cfg4", "tight16")})


if __name__ == "__main__":
    main()
