"""Plan searchers on the device: brute_force and random_search (ls/baselines.py:63-87,230-282),
plus greedy / genetic / heuristic_first_layer / homogeneous (ls/baselines.py:90-228).

Both keep the reference's signature, cap, tie rules and returned ScoredPlan. The sweep runs on
the device kernels (in-kernel plan decode / generation + per-plan scoring + (cost, rank)
argmin); with ``torch.distributed`` initialised the enumeration is dealt round-robin (rank r
sweeps indices r, r + W, r + 2W, ...: ``shard_strided``), the random-plan stream is split into
contiguous slices (``shard_range``; the PCG64 stream is jumped in-kernel), and the per-rank
winners meet in ONE all_gather of 48-byte keys — the only exchange the path has
(SURVEY.md §8(e)).
"""

from __future__ import annotations

import numpy as np

from . import _abi
from dataclasses import dataclass
from typing import Sequence

from .errors import ConfigError, InfeasibleError, InvariantError, PlanValidationError
from .instance import argmin_from_bytes, pcg_from_generator
from .model import ProvisionerConfig, ScoredPlan, SchedulingPlan
from .scoring import PlanScorer, device_instance

DEFAULT_ENUMERATION_CAP = 2 ** 24  # ls/baselines.py:27


def decode_index(index: int, num_types: int, num_layers: int) -> tuple:
    """itertools.product order: layer 0 is the most significant base-T digit."""
    digits = []
    for _ in range(num_layers):
        index, d = divmod(index, num_types)
        digits.append(d)
    return tuple(reversed(digits))


def decode_packed(rank: int, num_types: int, num_layers: int) -> tuple:
    """Inverse of the packed lexicographic rank (ceil(log2 T) bits per layer)."""
    bits = max(1, (num_types - 1).bit_length())
    mask = (1 << bits) - 1
    return tuple((rank >> ((num_layers - 1 - l) * bits)) & mask for l in range(num_layers))


def shard_range(begin: int, end: int, rank: int, world: int) -> tuple:
    """Contiguous shard r of [begin, end) (SURVEY.md §8(e) partitioning)."""
    n = end - begin
    return begin + n * rank // world, begin + n * (rank + 1) // world


def shard_strided(begin: int, end: int, rank: int, world: int) -> tuple:
    """Rank r's indices of [begin, end) as (first, stride, count): every world-th plan.
    Provisioning work is correlated between neighbouring plans (they share their leading
    layers' stages), so contiguous shards differ by up to 25% in sweep time at 4 GPUs;
    dealing single plans round-robin balances them."""
    n = end - begin
    count = (n - rank + world - 1) // world if n > rank else 0
    return begin + rank, world, count


def enum_shard_async(inst, begin: int, end: int, rank: int, world: int,
                     feasible_only: bool = True, stream=None):
    """This rank's argmin key over its strided shard of [begin, end)."""
    if world == 1:
        return inst.enum_argmin_async(begin, end, feasible_only, stream)
    first, stride, count = shard_strided(begin, end, rank, world)
    return inst.enum_argmin_strided_async(first, stride, count, feasible_only, stream)


def _dist():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist
    except ImportError:  # pragma: no cover
        pass
    return None


def merge_keys(keys: list) -> dict:
    """Deterministic min over per-rank argmin keys: (cost, rank); sums the counters."""
    best = None
    for k in keys:
        if best is None or (k["cost"], k["rank"]) < (best["cost"], best["rank"]):
            best = dict(k)
    best["evaluated"] = sum(k["evaluated"] for k in keys)
    best["feasible"] = sum(k["feasible"] for k in keys)
    best["flags"] = 0
    for k in keys:
        best["flags"] |= k["flags"]
    return best


def _split_keys(raw: bytes) -> list:
    n = _abi.ARGMIN_NBYTES
    return [argmin_from_bytes(raw[i:i + n]) for i in range(0, len(raw), n)]


def allgather_argmin(buf, group=None) -> dict:
    """One all_gather of the 48-byte device keys (one or more per rank, the same count on
    every rank), then the deterministic host merge."""
    dist = _dist()
    if dist is None or dist.get_world_size(group) == 1:
        keys = _split_keys(bytes(buf.cpu().numpy().tobytes()))
        return keys[0] if len(keys) == 1 else merge_keys(keys)
    import torch
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty(world * buf.numel(), dtype=torch.uint8, device=buf.device)
        dist.all_gather_into_tensor(out, buf, group=group)
        raw = out.cpu().numpy().tobytes()
    else:
        cpu = buf.cpu()
        outs = [torch.empty_like(cpu) for _ in range(world)]
        dist.all_gather(outs, cpu, group=group)
        raw = b"".join(o.numpy().tobytes() for o in outs)
    return merge_keys(_split_keys(raw))


def _raise_flags(key: dict):
    if key["flags"] & 2:
        raise PlanValidationError("a plan uses a type id or layer profile the instance lacks")
    if key["flags"] & 1:
        raise InvariantError("catalog has no CPU-capable resource type")


def enumerate_argmin(graph, catalog, params, begin: int, end: int, feasible_only: bool = True,
                     config: ProvisionerConfig = ProvisionerConfig(), group=None) -> dict:
    """Sharded enumeration argmin over [begin, end); every rank gets the merged key."""
    dist = _dist()
    rank, world = (dist.get_rank(group), dist.get_world_size(group)) if dist else (0, 1)
    inst = device_instance(graph, catalog, params, config)
    buf = enum_shard_async(inst, begin, end, rank, world, feasible_only)
    return allgather_argmin(buf, group)


def brute_force(graph, catalog, params, config: ProvisionerConfig = ProvisionerConfig(),
                enumeration_cap: int = DEFAULT_ENUMERATION_CAP, group=None,
                prune: bool = False) -> ScoredPlan:
    """Cheapest feasible plan over all T^L assignments (ls/baselines.py:63-87).

    ``prune=True`` (one GPU) skips index ranges whose certified cost lower bound exceeds an
    incumbent (hps_enum_argmin_pruned): the same plan, cost and tie-breaking, fewer plans scored.
    Instances it does not apply to (no CPU type, unprofiled layers) and multi-rank runs sweep
    everything."""
    T, L = catalog.num_types, graph.num_layers
    total = T ** L
    if total > enumeration_cap:
        raise ConfigError(f"brute force would enumerate {total} plans ({T}^{L}), "
                          f"cap is {enumeration_cap}")
    key = None
    dist = _dist()
    if prune and L > 1 and (dist is None or dist.get_world_size(group) == 1):
        try:
            key, _ = device_instance(graph, catalog, params, config).enum_argmin_pruned()
        except ConfigError:
            key = None
    if key is None:
        key = enumerate_argmin(graph, catalog, params, 0, total, True, config, group)
    _raise_flags(key)
    if not key["cost"] < float("inf"):
        raise InfeasibleError(f"no feasible plan among {total} enumerated")
    best = PlanScorer(graph, catalog, params, config)(SchedulingPlan(decode_index(key["rank"], T, L)))
    if best.cost != key["cost"]:  # the winner is re-scored through the same kernel
        raise InvariantError("winner re-score disagrees with the sweep")
    return ScoredPlan(best.plan, best.provisioning, best.cost, best.report, total)


def random_search(graph, catalog, params, budget: int, seed: int = 0, dedup: bool = False,
                  config: ProvisionerConfig = ProvisionerConfig(), group=None) -> ScoredPlan:
    """Best of ``budget`` random plans, penalties included (ls/baselines.py:230-282)."""
    if budget < 1:
        raise ConfigError("random search budget must be >= 1")
    T, L = catalog.num_types, graph.num_layers
    rng = np.random.default_rng(seed)
    inst = device_instance(graph, catalog, params, config)
    dist = _dist()
    rank, world = (dist.get_rank(group), dist.get_world_size(group)) if dist else (0, 1)
    if not dedup and T & (T - 1) == 0 and (max(1, (T - 1).bit_length()) * L) <= 128:
        # plans generated in-kernel from the generator's PCG64 stream
        lo, hi = shard_range(0, budget, rank, world)
        key = allgather_argmin(inst.random_argmin_async(pcg_from_generator(rng), lo, hi - lo), group)
        count = budget
    else:
        # the assignment list is the reference's own RNG stream (ls/baselines.py:252-272)
        assignments = _reference_assignments(rng, T, L, budget, dedup)
        import torch
        arr = torch.from_numpy(np.array(assignments, dtype=np.uint8).reshape(len(assignments), L))
        lo, hi = shard_range(0, len(assignments), rank, world)
        key = allgather_argmin(inst.plans_argmin_async(arr[lo:hi], feasible_only=False), group)
        count = len(assignments)
    _raise_flags(key)
    winner = decode_packed(key["rank"], T, L) if T > 1 else (0,) * L
    best = PlanScorer(graph, catalog, params, config)(SchedulingPlan(winner))
    return ScoredPlan(best.plan, best.provisioning, best.cost, best.report, count)


def _reference_assignments(rng, T, L, budget, dedup):
    total = T ** L
    if dedup and total <= 2 ** 20:
        chosen = rng.permutation(total)[:min(budget, total)]
        return [decode_index(int(c), T, L) for c in chosen]
    if dedup:
        seen, attempts = set(), 0
        while len(seen) < budget and attempts < 20 * budget:
            seen.add(tuple(int(g) for g in rng.integers(0, T, L)))
            attempts += 1
        return sorted(seen)
    return [tuple(int(g) for g in rng.integers(0, T, L)) for _ in range(budget)]


def _better(candidate, incumbent) -> bool:
    """Strictly cheaper, or equally cheap with a lexicographically smaller plan
    (ls/baselines.py:54-60)."""
    if incumbent is None:
        return True
    if candidate.cost != incumbent.cost:
        return candidate.cost < incumbent.cost
    return candidate.plan.assignment < incumbent.plan.assignment


def greedy(graph, catalog, params, config: ProvisionerConfig = ProvisionerConfig()) -> ScoredPlan:
    """Left-to-right layer fixing with suffix fill (ls/baselines.py:90-117). The T candidates of
    each layer are one device batch; ties go to the lower type id."""
    T, L = catalog.num_types, graph.num_layers
    scorer = PlanScorer(graph, catalog, params, config)
    decided: list = []
    for _ in range(L):
        cands = [tuple(decided) + (t,) * (L - len(decided)) for t in range(T)]
        scored = scorer.score_many(cands)
        best_type, best = 0, None
        for t, sc in enumerate(scored):
            if best is None or sc.cost < best.cost:
                best, best_type = sc, t
        decided.append(best_type)
    final = scorer(SchedulingPlan(tuple(decided)))
    return ScoredPlan(final.plan, final.provisioning, final.cost, final.report, scorer.evaluations)


@dataclass(frozen=True)
class GeneticConfig:
    """Genetic-search knobs (ls/baselines.py:30-51); ``mutation_rate=None`` means 1/L."""
    population: int = 64
    generations: int = 200
    crossover_rate: float = 0.8
    mutation_rate: float | None = None
    tournament_size: int = 3
    seed: int = 0

    def __post_init__(self):
        if self.population < 2:
            raise InvariantError("population must be >= 2")
        if not 0.0 <= self.crossover_rate <= 1.0:
            raise InvariantError("crossover_rate must be in [0, 1]")
        if self.mutation_rate is not None and not 0.0 <= self.mutation_rate <= 1.0:
            raise InvariantError("mutation_rate must be in [0, 1]")
        if self.tournament_size < 1:
            raise InvariantError("tournament_size must be >= 1")
        if self.generations < 0:
            raise InvariantError("generations must be >= 0")


def genetic(graph, catalog, params, config: GeneticConfig = GeneticConfig(),
            provisioner_config: ProvisionerConfig = ProvisionerConfig(),
            seed_plans: Sequence = ()) -> ScoredPlan:
    """Tournament selection, one-point crossover, per-gene mutation, one elite
    (ls/baselines.py:120-187). The RNG draws are the reference's numpy Generator calls in the
    same order; each generation's population is scored as one device batch."""
    T, L = catalog.num_types, graph.num_layers
    mutation_rate = config.mutation_rate if config.mutation_rate is not None else 1.0 / L
    rng = np.random.default_rng(config.seed)
    scorer = PlanScorer(graph, catalog, params, provisioner_config)
    population = [p.assignment for p in seed_plans][:config.population]
    while len(population) < config.population:
        population.append(tuple(int(g) for g in rng.integers(0, T, L)))
    best = None

    def evaluate_population(pop):
        nonlocal best
        scored = scorer.score_many(pop)
        for sc in scored:
            if _better(sc, best):
                best = sc
        return scored

    scored = evaluate_population(population)
    for _ in range(config.generations):
        costs = np.array([sc.cost for sc in scored])
        children = [population[int(np.argmin(costs))]]
        while len(children) < config.population:
            parents = []
            for _ in range(2):
                entrants = rng.integers(0, len(population), config.tournament_size)
                winner = min(entrants, key=lambda i: (costs[i], i))
                parents.append(population[int(winner)])
            mother, father = parents
            if L > 1 and rng.random() < config.crossover_rate:
                point = int(rng.integers(1, L))
                child = mother[:point] + father[point:]
            else:
                child = mother
            genes = list(child)
            for g in range(L):
                if rng.random() < mutation_rate:
                    genes[g] = int(rng.integers(0, T))
            children.append(tuple(genes))
        population = children
        scored = evaluate_population(population)
    return ScoredPlan(best.plan, best.provisioning, best.cost, best.report, scorer.evaluations)


def heuristic_first_layer(graph, catalog, invert: bool = False) -> SchedulingPlan:
    """First layer on the cheapest CPU type, the rest on the accelerator with the smallest
    summed computation time; ``invert`` swaps the roles (ls/baselines.py:190-219)."""
    cpu = catalog.cheapest_cpu_type()
    accelerators = [t for t in catalog.types if not t.is_cpu]

    def best_accel(layers) -> int:
        if not accelerators:
            raise ConfigError("heuristic needs at least one accelerator type")
        return min(accelerators,
                   key=lambda t: (sum(l.per_type_oct[t.id] for l in layers), t.id)).id

    if not invert:
        if graph.num_layers == 1:
            return SchedulingPlan((cpu.id,))
        gpu = best_accel(graph.layers[1:])
        return SchedulingPlan((cpu.id,) + (gpu,) * (graph.num_layers - 1))
    gpu = best_accel(graph.layers[:1])
    return SchedulingPlan((gpu,) + (cpu.id,) * (graph.num_layers - 1))


def homogeneous(graph, catalog, type_id: int) -> SchedulingPlan:
    """Every layer on one type (ls/baselines.py:222-228)."""
    if not 0 <= type_id < catalog.num_types:
        raise PlanValidationError(f"unknown type id {type_id} (catalog has "
                                  f"{catalog.num_types} types)")
    return SchedulingPlan((type_id,) * graph.num_layers)


__all__ = ["brute_force", "random_search", "greedy", "genetic", "GeneticConfig",
           "heuristic_first_layer", "homogeneous", "enumerate_argmin", "allgather_argmin", "merge_keys",
           "shard_range", "shard_strided", "enum_shard_async", "decode_index", "decode_packed", "DEFAULT_ENUMERATION_CAP"]
