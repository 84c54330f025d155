"""Domain types of the plan evaluator.

Field names, invariants and error classes follow the reference so its users can pass the
same objects (or the reference's own objects — everything here is read by attribute name):
  LayerSpec/ModelGraph/ResourceType/ResourceCatalog/SchedulingPlan/Stage/ProvisioningPlan/
  CostReport  ls/domain.py:21-252
  JobParams   ls/costmodel.py:39-47
  ProvisionerConfig ls/provisioner.py:57-72
  ScoredPlan  ls/scoring.py:27-44
The numeric work (stage aggregation, provisioning, cost) is NOT here: it runs in the CUDA
library (paper_2111_10635_b200/csrc), reached through ``instance.DeviceInstance``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Mapping

from .errors import InvariantError

SECONDS_PER_HOUR = 3600.0
PENALTY_FACTOR = 1e6          # ls/scoring.py:24
BREAKPOINT_LIMIT = 4096       # ls/provisioner.py:49
MODE_OPTIMAL = "optimal"      # ls/provisioner.py:51-54
MODE_STARATIO = "staratio"
MODE_STAPSRATIO = "stapsratio"
PROVISIONING_MODES = (MODE_OPTIMAL, MODE_STARATIO, MODE_STAPSRATIO)
STATIC_CPU_PER_GPU = 6        # ls/provisioner.py:47


def _check_fraction(layer: int, name: str, table: Mapping[int, float]) -> None:
    bad = {t: v for t, v in table.items() if not (0.0 <= v <= 1.0)}
    if bad:
        t, v = next(iter(bad.items()))
        raise InvariantError(f"layer {layer}: {name}[{t}] must be in [0,1], got {v}")


@dataclass(frozen=True)
class LayerSpec:
    """Profiled layer: per-type compute (oct) / communication (odt) seconds and their
    parallelisable fractions (alpha / beta) at the profiling batch size."""

    index: int
    layer_kind: str
    input_size: float
    weight_size: float
    per_type_oct: Mapping[int, float]
    per_type_odt: Mapping[int, float]
    per_type_alpha: Mapping[int, float]
    per_type_beta: Mapping[int, float]

    def __post_init__(self):
        if self.index < 0:
            raise InvariantError(f"layer index must be >= 0, got {self.index}")
        if min(self.input_size, self.weight_size) < 0:
            raise InvariantError(f"layer {self.index}: input_size and weight_size must be >= 0")
        for name, table in (("oct", self.per_type_oct), ("odt", self.per_type_odt)):
            neg = [(t, v) for t, v in table.items() if v < 0]
            if neg:
                raise InvariantError(
                    f"layer {self.index}: {name}[{neg[0][0]}] must be >= 0, got {neg[0][1]}")
        _check_fraction(self.index, "alpha", self.per_type_alpha)
        _check_fraction(self.index, "beta", self.per_type_beta)

    def covers_types(self, type_ids) -> bool:
        tables = (self.per_type_oct, self.per_type_odt, self.per_type_alpha, self.per_type_beta)
        return all(t in tab for tab in tables for t in type_ids)


@dataclass(frozen=True)
class ModelGraph:
    """Linear layer chain plus job counts: M (total_samples), epochs, B, B_o."""

    name: str
    layers: tuple
    total_samples: int
    epochs: int
    batch_size: int
    profile_batch_size: int

    def __post_init__(self):
        object.__setattr__(self, "layers", tuple(self.layers))
        if len(self.layers) == 0:
            raise InvariantError("model graph must have at least one layer")
        for pos, layer in enumerate(self.layers):
            if layer.index != pos:
                raise InvariantError(
                    f"layer indices must be contiguous from 0; position {pos} holds index {layer.index}")
        checks = ((self.profile_batch_size >= 1, "profile_batch_size must be >= 1"),
                  (self.batch_size >= 1, "batch_size must be >= 1"),
                  (self.total_samples >= self.batch_size, "total_samples must be >= batch_size"),
                  (self.epochs >= 1, "epochs must be >= 1"))
        for ok, msg in checks:
            if not ok:
                raise InvariantError(msg)

    @property
    def num_layers(self) -> int:
        return len(self.layers)


@dataclass(frozen=True)
class ResourceType:
    id: int
    name: str
    price_per_hour: float
    unit: str
    quota: int
    is_cpu: bool

    def __post_init__(self):
        if not self.price_per_hour > 0:
            raise InvariantError(f"type {self.id} ({self.name}): price_per_hour must be > 0")
        if self.quota < 1:
            raise InvariantError(f"type {self.id} ({self.name}): quota must be >= 1")


@dataclass(frozen=True)
class ResourceCatalog:
    types: tuple
    layer_kinds: tuple = ()

    def __post_init__(self):
        object.__setattr__(self, "types", tuple(self.types))
        object.__setattr__(self, "layer_kinds", tuple(self.layer_kinds))
        if not self.types:
            raise InvariantError("catalog must declare at least one resource type")
        ids = [t.id for t in self.types]
        if ids != list(range(len(ids))):
            raise InvariantError(f"type ids must be unique and contiguous from 0, got {ids}")

    @property
    def num_types(self) -> int:
        return len(self.types)

    def cheapest_cpu_type(self) -> ResourceType:
        """Cheapest CPU-capable type, lowest id on a price tie (ls/domain.py:163-167)."""
        cpus = sorted((t for t in self.types if t.is_cpu), key=lambda t: (t.price_per_hour, t.id))
        if not cpus:
            raise InvariantError("catalog has no CPU-capable resource type")
        return cpus[0]


@dataclass(frozen=True)
class SchedulingPlan:
    """``assignment[l]`` = resource type id of layer l."""

    assignment: tuple

    def __post_init__(self):
        object.__setattr__(self, "assignment", tuple(int(a) for a in self.assignment))
        if not self.assignment:
            raise InvariantError("scheduling plan must cover at least one layer")

    def __len__(self) -> int:
        return len(self.assignment)


@dataclass(frozen=True)
class Stage:
    index: int
    type_id: int
    layer_range: tuple
    oct: float
    odt: float
    alpha: float
    beta: float

    @property
    def num_layers(self) -> int:
        return self.layer_range[1] - self.layer_range[0] + 1


@dataclass(frozen=True)
class ProvisioningPlan:
    per_stage_k: tuple
    ps_cores: int
    per_type_totals: Mapping[int, int]

    def __post_init__(self):
        object.__setattr__(self, "per_stage_k", tuple(int(k) for k in self.per_stage_k))
        object.__setattr__(self, "per_type_totals", dict(self.per_type_totals))
        if any(k < 1 for k in self.per_stage_k):
            raise InvariantError("every per-stage count must be >= 1")
        if self.ps_cores < 0:
            raise InvariantError("ps_cores must be >= 0")

    @property
    def total_units(self) -> int:
        return sum(self.per_type_totals.values())


@dataclass(frozen=True)
class CostReport:
    per_stage_ct: tuple
    per_stage_dt: tuple
    per_stage_et: tuple
    per_stage_throughput: tuple
    pipeline_throughput: float
    total_exec_time: float
    monetary_cost: float
    feasible: bool
    violation: str | None = None


@dataclass(frozen=True)
class JobParams:
    throughput_limit: float

    def __post_init__(self):
        if not self.throughput_limit > 0:
            raise InvariantError("throughput_limit must be > 0")


@dataclass(frozen=True)
class ProvisionerConfig:
    ps_cores_per_gpu: float = 6.0
    newton_max_iters: int = 50
    newton_tol: float = 1e-3
    fd_step: float = 1e-3

    def __post_init__(self):
        if min(self.ps_cores_per_gpu, self.newton_max_iters, self.newton_tol, self.fd_step) <= 0:
            raise InvariantError("all provisioner parameters must be positive")


@dataclass(frozen=True)
class ScoredPlan:
    """A plan, its provisioning (None when infeasible) and its cost (or penalty)."""

    plan: SchedulingPlan
    provisioning: ProvisioningPlan | None
    cost: float
    report: CostReport | None = None
    evaluations: int | None = None

    @property
    def feasible(self) -> bool:
        return self.provisioning is not None


def penalty_cost(catalog, gap: float) -> float:
    """Penalty of an infeasible plan: 1e6 x the top hourly price x (1 + gap)
    (ls/scoring.py:47-50). Host-side scalar used only to label single plans; the kernels
    compute the same expression for every plan they score."""
    top = max(t.price_per_hour for t in catalog.types)
    return PENALTY_FACTOR * top * (1.0 + max(0.0, gap))
