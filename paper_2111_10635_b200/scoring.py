"""Drop-in scoring API: PlanScorer, provision, optimize_k1, evaluate, build_stages.

Signatures and return types follow the reference (ls/scoring.py:53-101,
ls/provisioner.py:374-584, ls/costmodel.py:102-167, ls/domain.py:255-328); every number comes
from the CUDA library through :class:`~.instance.DeviceInstance`. The host only validates
arguments, assembles the reference's dataclasses and maps status bytes to exceptions.
"""

from __future__ import annotations

from collections import OrderedDict

import numpy as np

from . import _abi
from .errors import InfeasibleError, InvariantError, PlanValidationError
from .model import (MODE_OPTIMAL, MODE_STAPSRATIO, MODE_STARATIO, PROVISIONING_MODES, STATIC_CPU_PER_GPU, CostReport, JobParams, ProvisionerConfig,
                    ProvisioningPlan, ResourceCatalog, ResourceType, ScoredPlan, SchedulingPlan,
                    Stage, penalty_cost)

_MESSAGES = {
    _abi.ST_MIN_K1: "stage 0 cannot reach the throughput limit at any count: serial time "
                    "exceeds the budget",
    _abi.ST_SERIAL: "a stage cannot reach the throughput limit at any count: its serial time "
                    "is not below the budget",
    _abi.ST_QUOTA_TAU_HI: "no count within quota meets the throughput limit: a type needs more "
                          "units than its quota",
    _abi.ST_FLOOR_TAU_HI: "a stage cannot reach the load-balance target at any count",
    _abi.ST_NO_CANDIDATE: "no count within quota meets the throughput limit strictly",
    _abi.ST_PS_QUOTA: "the CPU type cannot host the parameter-server cores within its quota",
    _abi.ST_STATIC_NONE: "no ratio multiple within quota meets the throughput limit",
}

_INSTANCES: "OrderedDict[tuple, object]" = OrderedDict()
_MAX_CACHED = 8


def device_instance(graph, catalog, job, config=None, with_ps=True):
    """Cached DeviceInstance for (graph, catalog, job, config, with_ps) on the current device."""
    import torch
    from .instance import DeviceInstance

    config = config if config is not None else ProvisionerConfig()
    dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
    key = (id(graph), id(catalog), float(job.throughput_limit), config, bool(with_ps), dev)
    inst = _INSTANCES.get(key)
    if inst is not None and inst.graph is graph and inst.catalog is catalog:
        _INSTANCES.move_to_end(key)
        return inst
    inst = DeviceInstance(graph, catalog, job, config, with_ps)
    _INSTANCES[key] = inst
    while len(_INSTANCES) > _MAX_CACHED:
        _INSTANCES.popitem(last=False)
    return inst


def validate_plan(plan, graph, catalog) -> None:
    """Length and id checks of ls/domain.py:255-272 (pure argument validation)."""
    if len(plan.assignment) != graph.num_layers:
        raise PlanValidationError(f"plan covers {len(plan.assignment)} layers but model "
                                  f"'{graph.name}' has {graph.num_layers}")
    for l, t in enumerate(plan.assignment):
        if not 0 <= t < catalog.num_types:
            raise PlanValidationError(f"layer {l} assigned to unknown type id {t} "
                                      f"(catalog has {catalog.num_types} types)")


def _runs(assignment):
    """(type, first, last) of each maximal run — index bookkeeping only."""
    out, start = [], 0
    for pos in range(1, len(assignment) + 1):
        if pos == len(assignment) or assignment[pos] != assignment[start]:
            out.append((assignment[start], start, pos - 1))
            start = pos
    return out


def _totals(runs, k, ps, ps_type):
    totals: dict[int, int] = {}
    for (t, _, _), kk in zip(runs, k):
        totals[t] = totals.get(t, 0) + int(kk)
    if ps > 0:
        totals[ps_type] = totals.get(ps_type, 0) + int(ps)
    return totals


def infeasible_message(code: int, ex, catalog) -> str:
    """The reference's InfeasibleError text for a device status and its hps_explain details
    (ls/provisioner.py:98-101, 164-174, 407-411, 421-425, 473-477, 508-511)."""
    label = ("computation", "communication")
    if code == _abi.ST_MIN_K1:
        return (f"stage {ex.stage} cannot reach the throughput limit at any count: serial "
                f"{label[ex.side]} time exceeds the budget")
    if code == _abi.ST_SERIAL:
        return (f"stage {ex.stage} cannot reach the throughput limit at any count: its serial "
                f"time {ex.serial:.6g}s is not below the budget {ex.tau_hi:.6g}s")
    if code == _abi.ST_FLOOR_TAU_HI:
        if ex.serial_side:
            return f"stage {ex.stage}: serial {label[ex.side]} time exceeds the load-balance target"
        return f"stage {ex.stage}: {label[ex.side]} cannot reach the load-balance target at any count"
    if code == _abi.ST_QUOTA_TAU_HI:
        rt = catalog.types[ex.type]
        units = (ex.units_hi << 64) | ex.units_lo
        return (f"no count within quota meets the throughput limit: type '{rt.name}' needs "
                f"{units} units, quota is {rt.quota}")
    if code == _abi.ST_PS_QUOTA:
        rt = catalog.types[ex.type]
        return (f"type '{rt.name}' needs {ex.units_lo} units including {ex.ps} parameter-server "
                f"cores, quota is {rt.quota}")
    return _MESSAGES.get(code, "infeasible plan")


def raise_for_status(code: int, gap: float) -> None:
    if code == _abi.ST_OK:
        return
    if code == _abi.ST_INVALID:
        raise PlanValidationError("plan uses a type id or layer profile the instance lacks")
    if code == _abi.ST_NO_CPU_TYPE:
        raise InvariantError("catalog has no CPU-capable resource type")
    raise InfeasibleError(_MESSAGES.get(code, "infeasible plan"), gap=gap)


class PlanScorer:
    """Callable scoring plans for one (graph, catalog, job) instance (ls/scoring.py:53-101).

    Results are cached by assignment like the reference; ``evaluations`` counts distinct
    plans scored. :meth:`score_many` scores a whole batch in one kernel launch and
    :meth:`score_arrays` returns the raw device tensors (no Python objects per plan).
    """

    def __init__(self, graph, catalog, params, config: ProvisionerConfig = ProvisionerConfig(),
                 mode: str = MODE_OPTIMAL, with_ps: bool = True):
        if mode not in PROVISIONING_MODES:
            raise InvariantError(f"unknown provisioning mode '{mode}'")
        self.graph, self.catalog, self.params, self.config = graph, catalog, params, config
        self.mode, self.with_ps = mode, with_ps
        self.evaluations = 0
        self._cache: dict[tuple, ScoredPlan] = {}
        self._inst = None

    @property
    def instance(self):
        if self._inst is None:
            self._inst = device_instance(self.graph, self.catalog, self.params, self.config,
                                         self.with_ps)
        return self._inst

    def __call__(self, plan) -> ScoredPlan:
        hit = self._cache.get(plan.assignment)
        if hit is not None:
            return hit
        return self.score_many([plan])[0]

    def score_arrays(self, plans_u8, want_k: bool = True):
        """Batched device scoring; ``plans_u8`` is a uint8 [n, L] array or tensor."""
        import torch
        if not torch.is_tensor(plans_u8):
            plans_u8 = torch.from_numpy(np.ascontiguousarray(plans_u8, dtype=np.uint8))
        return self.instance.score(plans_u8.to(self.instance.device), want_k=want_k,
                                   mode=self.mode, cpu_per_gpu=STATIC_CPU_PER_GPU)

    def score_many(self, plans) -> list:
        import torch
        plans = [p if isinstance(p, SchedulingPlan) or hasattr(p, "assignment")
                 else SchedulingPlan(tuple(p)) for p in plans]
        todo = [p for p in dict.fromkeys(p.assignment for p in plans) if p not in self._cache]
        for a in todo:
            validate_plan(SchedulingPlan(a), self.graph, self.catalog)
        if todo:
            arr = torch.tensor(np.array(todo, dtype=np.uint8).reshape(len(todo), -1))
            out = self.score_arrays(arr)
            host = {k: v.cpu().numpy() for k, v in out.items() if v is not None}
            ok_rows = [i for i in range(len(todo)) if host["status"][i] & _abi.ST_CODE_MASK == 0]
            reports = self._reports(arr, out, ok_rows) if ok_rows else {}
            for i, a in enumerate(todo):
                code = int(host["status"][i]) & _abi.ST_CODE_MASK
                if code in (_abi.ST_INVALID, _abi.ST_NO_CPU_TYPE):
                    raise_for_status(code, 0.0)
                plan = SchedulingPlan(a)
                if code == _abi.ST_OK:
                    S = int(host["num_stages"][i])
                    k = tuple(int(x) for x in host["k"][i, :S])
                    ps = int(host["ps"][i])
                    runs = _runs(a)
                    ps_type = (self.catalog.cheapest_cpu_type().id if ps > 0 else None)
                    prov = ProvisioningPlan(k, ps, _totals(runs, k, ps, ps_type))
                    scored = ScoredPlan(plan, prov, float(host["cost"][i]), reports[i])
                else:
                    scored = ScoredPlan(plan, None, float(host["cost"][i]), None)
                self._cache[a] = scored
                self.evaluations += 1
        return [self._cache[p.assignment] for p in plans]

    def _reports(self, arr, out, rows):
        import torch
        inst = self.instance
        idx = torch.tensor(rows, dtype=torch.long, device=inst.device)
        rep = inst.report(arr.to(inst.device)[idx], out["k"][idx], out["ps"][idx])
        host = {k: v.cpu().numpy() for k, v in rep.items()}
        res = {}
        for j, i in enumerate(rows):
            S = int(out["num_stages"][i].item())
            res[i] = CostReport(
                per_stage_ct=tuple(float(x) for x in host["ct"][j, :S]),
                per_stage_dt=tuple(float(x) for x in host["dt"][j, :S]),
                per_stage_et=tuple(float(x) for x in host["et"][j, :S]),
                per_stage_throughput=tuple(float(x) for x in host["tp"][j, :S]),
                pipeline_throughput=float(host["pipeline_tp"][j]),
                total_exec_time=float(host["exec_time"][j]),
                monetary_cost=float(host["cost"][j]),
                feasible=bool(host["feasible"][j]), violation=None)
        return res


def provision(plan, graph, catalog, params, config: ProvisionerConfig = ProvisionerConfig(),
              mode: str = MODE_OPTIMAL, with_ps: bool = True) -> ProvisioningPlan:
    """ls/provisioner.py:564-584 on the device; raises InfeasibleError(gap) like the reference.

    ``mode`` 'staratio' / 'stapsratio' dispatches to static_provision (ls/provisioner.py:516-561).
    """
    if mode not in PROVISIONING_MODES:
        raise InvariantError(f"unknown provisioning mode '{mode}'")
    validate_plan(plan, graph, catalog)
    import torch
    inst = device_instance(graph, catalog, params, config, with_ps)
    out = inst.score(torch.tensor([list(plan.assignment)], dtype=torch.uint8), mode=mode,
                     cpu_per_gpu=STATIC_CPU_PER_GPU)
    return _provisioning_from(out, plan, graph, catalog, params, inst, mode, STATIC_CPU_PER_GPU)


def static_provision(plan, graph, catalog, params, mode: str,
                     cpu_per_gpu: int = STATIC_CPU_PER_GPU) -> ProvisioningPlan:
    """Fixed-ratio provisioning baseline (ls/provisioner.py:516-561) on the device."""
    if mode not in (MODE_STARATIO, MODE_STAPSRATIO):
        raise InvariantError(f"unknown static provisioning mode '{mode}'")
    validate_plan(plan, graph, catalog)
    import torch
    inst = device_instance(graph, catalog, params)
    out = inst.score(torch.tensor([list(plan.assignment)], dtype=torch.uint8), mode=mode,
                     cpu_per_gpu=cpu_per_gpu)
    return _provisioning_from(out, plan, graph, catalog, params, inst, mode, cpu_per_gpu)


def _static_violation(plan, catalog, params, inst, mode, cpu_per_gpu):
    """The reference's InfeasibleError text carries the last scanned multiplier's violation
    (ls/provisioner.py:553-561). The scan's last g is the quota bound g_max (integer
    bookkeeping here); its throughput comes from the device evaluate()."""
    import torch
    runs = _runs(plan.assignment)
    f = [cpu_per_gpu if catalog.types[t].is_cpu else 1 for t, _, _ in runs]
    n_acc = sum(1 for t, _, _ in runs if not catalog.types[t].is_cpu)
    per = {}
    for (t, _, _), x in zip(runs, f):
        per[t] = per.get(t, 0) + x
    ps_per = cpu_per_gpu * n_acc if mode == MODE_STAPSRATIO else 0
    if ps_per > 0:
        cpu = catalog.cheapest_cpu_type().id
        per[cpu] = per.get(cpu, 0) + ps_per
    gmax = min(max(t.quota for t in catalog.types),
               *(catalog.types[t].quota // m for t, m in per.items()))
    if gmax < 1:
        return None
    k = torch.zeros((1, len(plan.assignment)), dtype=torch.int32)
    k[0, :len(runs)] = torch.tensor([x * gmax for x in f], dtype=torch.int32)
    rep = inst.report(torch.tensor([list(plan.assignment)], dtype=torch.uint8), k,
                      torch.tensor([ps_per * gmax], dtype=torch.int32))
    overall = float(rep["pipeline_tp"][0].item())
    return (f"pipeline throughput {overall:.6g} does not strictly exceed "
            f"limit {params.throughput_limit:.6g}")


def _provisioning_from(out, plan, graph, catalog, params, inst, mode, cpu_per_gpu):
    code = int(out["status"][0].item()) & _abi.ST_CODE_MASK
    if code == _abi.ST_STATIC_NONE:
        last = _static_violation(plan, catalog, params, inst, mode, cpu_per_gpu)
        raise InfeasibleError(_MESSAGES[code] + (f": {last}" if last else ""), gap=1.0)
    if code not in (_abi.ST_OK, _abi.ST_INVALID, _abi.ST_NO_CPU_TYPE):
        import torch
        ex = inst.explain(torch.tensor([list(plan.assignment)], dtype=torch.uint8),
                          out["status"], out["k"])[0]
        raise InfeasibleError(infeasible_message(code, ex, catalog), gap=float(out["gap"][0].item()))
    raise_for_status(code, float(out["gap"][0].item()))
    S = int(out["num_stages"][0].item())
    k = tuple(int(x) for x in out["k"][0, :S].cpu().tolist())
    ps = int(out["ps"][0].item())
    ps_type = catalog.cheapest_cpu_type().id if ps > 0 else None
    return ProvisioningPlan(k, ps, _totals(_runs(plan.assignment), k, ps, ps_type))


def optimize_k1(plan, graph, catalog, params, config: ProvisionerConfig = ProvisionerConfig()):
    """Counts without parameter-server cores (ls/provisioner.py:374-483)."""
    return provision(plan, graph, catalog, params, config, MODE_OPTIMAL, with_ps=False)


def evaluate(plan, provisioning, graph, catalog, params) -> CostReport:
    """ls/costmodel.py:102-167: times, throughput and cost of given counts, on the device."""
    import torch
    validate_plan(plan, graph, catalog)
    runs = _runs(plan.assignment)
    if len(provisioning.per_stage_k) != len(runs):
        raise PlanValidationError(f"provisioning has {len(provisioning.per_stage_k)} stage "
                                  f"counts but the plan induces {len(runs)} stages")
    if any(k < 1 for k in provisioning.per_stage_k):
        raise InvariantError("resource count must be >= 1")
    inst = device_instance(graph, catalog, params)
    L = graph.num_layers
    k = torch.zeros((1, L), dtype=torch.int32)
    k[0, :len(runs)] = torch.tensor(provisioning.per_stage_k, dtype=torch.int32)
    rep = inst.report(torch.tensor([list(plan.assignment)], dtype=torch.uint8), k,
                      torch.tensor([provisioning.ps_cores], dtype=torch.int32))
    h = {n: v.cpu().numpy() for n, v in rep.items()}
    S = len(runs)
    overall = float(h["pipeline_tp"][0])
    violation = None
    if not overall > params.throughput_limit:
        violation = (f"pipeline throughput {overall:.6g} does not strictly exceed "
                     f"limit {params.throughput_limit:.6g}")
    else:
        for t in sorted(provisioning.per_type_totals):
            total, rt = provisioning.per_type_totals[t], catalog.types[t]
            if total > rt.quota:
                violation = f"type '{rt.name}' needs {total} units, quota is {rt.quota}"
                break
    return CostReport(
        per_stage_ct=tuple(float(x) for x in h["ct"][0, :S]),
        per_stage_dt=tuple(float(x) for x in h["dt"][0, :S]),
        per_stage_et=tuple(float(x) for x in h["et"][0, :S]),
        per_stage_throughput=tuple(float(x) for x in h["tp"][0, :S]),
        pipeline_throughput=overall, total_exec_time=float(h["exec_time"][0]),
        monetary_cost=float(h["cost"][0]), feasible=violation is None, violation=violation)


def build_stages(plan, graph) -> tuple:
    """Stages of a plan with the device stage table's aggregates (ls/domain.py:275-328)."""
    if len(plan.assignment) != graph.num_layers:
        raise PlanValidationError(f"plan covers {len(plan.assignment)} layers but model "
                                  f"'{graph.name}' has {graph.num_layers}")
    T = 1 + max(max(l.per_type_oct) for l in graph.layers)
    if max(plan.assignment) >= T:
        raise PlanValidationError("layer profiles do not cover the plan's type ids")
    cat = ResourceCatalog(tuple(ResourceType(t, f"t{t}", 1.0, "u", 1, True) for t in range(T)))
    inst = device_instance(graph, cat, JobParams(1.0))
    stages = []
    for i, (t, first, last) in enumerate(_runs(plan.assignment)):
        oct_, odt, alpha, beta = inst.stage_aggregates(t, first, last)
        stages.append(Stage(index=i, type_id=t, layer_range=(first, last), oct=oct_, odt=odt,
                            alpha=alpha, beta=beta))
    return tuple(stages)


__all__ = ["PlanScorer", "ScoredPlan", "penalty_cost", "provision", "static_provision",
           "optimize_k1", "evaluate",
           "build_stages", "validate_plan", "device_instance"]
