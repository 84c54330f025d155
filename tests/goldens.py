"""Helpers to read the committed golden records (generated from the reference)."""
from __future__ import annotations

import gzip
import json
from pathlib import Path

import numpy as np

from paper_2111_10635_b200 import graphio
from paper_2111_10635_b200.model import JobParams, ProvisionerConfig

GOLDEN = Path(__file__).resolve().parent / "golden"


def plan_from_str(s: str):
    return [int(ch, 36) for ch in s]


def read_jsonl(name: str):
    with gzip.open(GOLDEN / name, "rt") as f:
        return [json.loads(line) for line in f]


def instance(name: str):
    g, c, limit = graphio.load_fixture(name)
    return g, c, JobParams(limit)


def inline_instance(item: dict):
    g = graphio.graph_from_dict(item["graph"])
    c = graphio.catalog_from_dict(item["catalog"])
    return g, c, JobParams(item["throughput_limit"])


def plans_array(records) -> np.ndarray:
    return np.array([plan_from_str(r["plan"]) for r in records], dtype=np.uint8)


def staged(g, c, job, with_ps=True):
    from paper_2111_10635_b200._abi import StagedDesc
    return StagedDesc(g, c, job, ProvisionerConfig(), with_ps)


def expected(records):
    """Columns of a record list: cost (float64 from hex), status, gap, ps, k (ragged)."""
    cost = np.array([float.fromhex(r["cost"]) for r in records])
    status = np.array([r["status"] for r in records], dtype=np.int64)
    gap = np.array([float.fromhex(r["gap"]) if "gap" in r else 0.0 for r in records])
    ps = np.array([r.get("ps", 0) for r in records], dtype=np.int64)
    ovf = np.array([r.get("ovf", 0) for r in records], dtype=np.int64)
    return cost, status, gap, ps, ovf


PLAN_FILES = ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "quota", "tight16", "tightmn", "nce5", "emb2"]
