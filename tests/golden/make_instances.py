"""Freeze the BASELINE.json configurations as JSON fixtures (graph + catalog + limit).

Generated HERE by importing the reference package (``PYTHONPATH=/root/reference/pkg/src``);
the output travels with the repo so the GPU box never needs /root/reference.

Recipes follow SURVEY.md §8(d):
  cfg1  CTRDNN-4 = layers (0,2,3,4) of ctrdnn16, catalog_default, limit 5e4
  cfg2  MATCHNET-8 = matchnet16 layers[:8], 3-type variant catalog, limit 1e5
  cfg3  ctrdnn16, 3-type variant catalog, limit 5e4
  cfg4  ctrdnn16, catalog_default, limit 5e4
  cfg5  resize_model(ctrdnn16, 64), 4-type variant catalog, limit 5e4
plus edge instances used only by parity tests:
  quota   ctrdnn16 + catalog_quota_limited, limit 5e4
  tight16 ctrdnn16 + catalog_default, limit 1e4   (overflow path, >4096 breakpoints)
  tightmn matchnet16 + catalog_default, limit 1e4
  nce5    nce5 + 4-type variant catalog, limit 2e4
  emb2    emb2_10 + 3-type variant catalog, limit 5e4

Variant builders are ls/experiments.py:422-496 (resize_model, catalog_with_gpu_variants,
simulate_type_variants); run from this script, never copied.
"""
import json
import os
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import layersched as ls  # noqa: E402
from layersched import experiments as ex  # noqa: E402
from layersched.fileio import graph_to_dict, catalog_to_dict  # noqa: E402

OUT = Path(__file__).resolve().parent / "instances"


def sub_graph(graph, idx, name):
    layers = [replace(graph.layers[i], index=j) for j, i in enumerate(idx)]
    return replace(graph, name=name, layers=tuple(layers))


def variant(graph, catalog, t):
    cat = ex.catalog_with_gpu_variants(catalog, t)
    return ex.simulate_type_variants(graph, cat), cat


def build():
    ctr = ls.load_bundled_graph("ctrdnn16")
    mn = ls.load_bundled_graph("matchnet16")
    nce = ls.load_bundled_graph("nce5")
    emb = ls.load_bundled_graph("emb2_10")
    cat = ls.load_bundled_catalog("catalog_default")
    catq = ls.load_bundled_catalog("catalog_quota_limited")
    inst = {}
    inst["cfg1"] = (sub_graph(ctr, (0, 2, 3, 4), "ctrdnn4"), cat, 5e4)
    g, c = variant(sub_graph(mn, tuple(range(8)), "matchnet8"), cat, 3)
    inst["cfg2"] = (g, c, 1e5)
    g, c = variant(ctr, cat, 3)
    inst["cfg3"] = (g, c, 5e4)
    inst["cfg4"] = (ctr, cat, 5e4)
    g, c = variant(ex.resize_model(ctr, 64), cat, 4)
    inst["cfg5"] = (g, c, 5e4)
    inst["quota"] = (ctr, catq, 5e4)
    inst["tight16"] = (ctr, cat, 1e4)
    inst["tightmn"] = (mn, cat, 1e4)
    g, c = variant(nce, cat, 4)
    inst["nce5"] = (g, c, 2e4)
    g, c = variant(emb, cat, 3)
    inst["emb2"] = (g, c, 5e4)
    return inst


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    index = {}
    for name, (g, c, limit) in build().items():
        (OUT / f"{name}_graph.json").write_text(json.dumps(graph_to_dict(g), indent=1) + "\n")
        (OUT / f"{name}_catalog.json").write_text(json.dumps(catalog_to_dict(c), indent=1) + "\n")
        index[name] = {"graph": f"{name}_graph.json", "catalog": f"{name}_catalog.json",
                       "throughput_limit": limit, "layers": g.num_layers, "types": c.num_types}
    (OUT / "index.json").write_text(json.dumps(index, indent=1) + "\n")
    print(json.dumps(index, indent=1))


if __name__ == "__main__":
    main()
