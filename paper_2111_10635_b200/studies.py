"""provisioning_study (ls/experiments.py:626-703): compare provisioning modes on one plan.

Every number comes from the device (``scoring.provision`` / ``scoring.evaluate``); this module
only assembles rows and writes the reference's CSV layout.
"""
from __future__ import annotations

import csv
from dataclasses import dataclass
from pathlib import Path

from .errors import SchedulerError
from .model import PROVISIONING_MODES, ProvisionerConfig


@dataclass(frozen=True)
class ProvisioningRow:
    """ls/experiments.py:626-634."""
    mode: str
    cost: float | None
    throughput: float | None
    per_stage_k: tuple | None
    ps_cores: int | None
    feasible: bool
    error: str = ""


def _fmt(value) -> str:
    """CSV cell format of ls/experiments.py:304-311."""
    if value is None:
        return ""
    if isinstance(value, bool):
        return "true" if value else "false"
    if isinstance(value, float):
        return repr(value)
    return str(value)


def provisioning_study(plan, graph, catalog, job, modes=PROVISIONING_MODES,
                       provisioner_config: ProvisionerConfig = ProvisionerConfig(),
                       out_dir=None) -> list:
    """One row per mode; ``optimal`` without PS cores, like ls/experiments.py:646-651."""
    from .scoring import evaluate, provision
    rows = []
    for mode in modes:
        try:
            prov = provision(plan, graph, catalog, job, provisioner_config, mode=mode,
                             with_ps=False)
            rep = evaluate(plan, prov, graph, catalog, job)
            rows.append(ProvisioningRow(mode, rep.monetary_cost, rep.pipeline_throughput,
                                        prov.per_stage_k, prov.ps_cores, rep.feasible))
        except SchedulerError as exc:
            rows.append(ProvisioningRow(mode, None, None, None, None, False, str(exc)))
    if out_dir is not None:
        out_dir = Path(out_dir)
        out_dir.mkdir(parents=True, exist_ok=True)
        with open(out_dir / "provisioning.csv", "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(("mode", "cost", "throughput", "per_stage_k", "ps_cores", "feasible",
                        "error"))
            for r in rows:
                w.writerow([r.mode, _fmt(r.cost), _fmt(r.throughput),
                            "-".join(str(k) for k in r.per_stage_k) if r.per_stage_k else "",
                            _fmt(r.ps_cores), _fmt(r.feasible), r.error])
    return rows


__all__ = ["ProvisioningRow", "provisioning_study"]
