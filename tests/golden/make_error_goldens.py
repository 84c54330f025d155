"""InfeasibleError texts and gaps from the REFERENCE for every infeasibility class
(test infrastructure; run here only — the reference is importable in the build container).

    python tests/golden/make_error_goldens.py

Plans are drawn from the committed edge goldens (synth.jsonl.gz, c1.jsonl.gz: instances inline)
and the 'quota' / 'cfg2' fixtures, up to PER_CLASS per status class, and passed through the
reference's provision() (ls/provisioner.py:564-584; with_ps=False = optimize_k1). Each record
keeps the instance reference, the plan, with_ps, str(exc) and exc.gap as float.hex.
Output: tests/golden/errors.jsonl.gz (read by tests/test_gpu_errors.py).
"""
import gzip
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE))
import layersched as ls  # noqa: E402

import make_goldens as mg  # noqa: E402

PER_CLASS = 40


def _read(name):
    with gzip.open(HERE / name, "rt") as f:
        return [json.loads(line) for line in f]


def inline(item):
    with tempfile.TemporaryDirectory() as d:
        gp, cp = Path(d) / "g.json", Path(d) / "c.json"
        gp.write_text(json.dumps(item["graph"]))
        cp.write_text(json.dumps(item["catalog"]))
        return ls.load_model_graph(gp), ls.load_catalog(cp), ls.JobParams(item["throughput_limit"])


def main():
    rng = np.random.default_rng(11)
    pool = {}   # status -> [(src, item, plan)]
    for src in ("synth.jsonl.gz", "c1.jsonl.gz"):
        for i, it in enumerate(_read(src)):
            for r in it["records"]:
                if r["status"] not in (0, 255):
                    pool.setdefault(r["status"], []).append((src, i, r["plan"]))
    for name in ("quota", "cfg2"):
        for r in _read(f"plans_{name}.jsonl.gz"):
            if r["status"] != 0:
                pool.setdefault(r["status"], []).append((name, -1, r["plan"]))
    items = {src: _read(src) for src in ("synth.jsonl.gz", "c1.jsonl.gz")}
    cache = {}
    out = []
    for status in sorted(pool):
        cand = pool[status]
        pick = rng.choice(len(cand), size=min(PER_CLASS, len(cand)), replace=False)
        for j, p in enumerate(sorted(int(x) for x in pick)):
            src, i, plan_s = cand[p]
            key = (src, i)
            if key not in cache:
                cache[key] = inline(items[src][i]) if i >= 0 else mg.load_instance(src)
            g, c, job = cache[key]
            plan = ls.SchedulingPlan(tuple(int(ch, 36) for ch in plan_s))
            for with_ps in ((True, False) if j % 4 == 0 else (True,)):
                try:
                    ls.provision(plan, g, c, job, with_ps=with_ps)
                    continue   # (with_ps=False can make a PS-quota plan feasible)
                except ls.InfeasibleError as e:
                    out.append({"src": src, "item": i, "plan": plan_s, "with_ps": with_ps,
                                "status": status, "msg": str(e), "gap": e.gap.hex()})
    with gzip.open(HERE / "errors.jsonl.gz", "wt") as f:
        for r in out:
            f.write(json.dumps(r) + "\n")
    print(len(out), "records;", {s: sum(1 for r in out if r["status"] == s) for s in pool})


if __name__ == "__main__":
    main()
