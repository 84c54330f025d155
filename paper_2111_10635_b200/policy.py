"""Recurrent scheduling policy and its REINFORCE trainer on the device.

Drop-in for ``layersched.policy`` (ls/policy/features.py, network.py, training.py): the same
classes, field names, defaults and ``train`` signature. Per round the device runs the LSTM
forward (K4, FP64; the hoisted input projection on the FP64 tensor cores), samples all G plans
from the generator's PCG64 stream with numpy's exact ``Generator.choice`` arithmetic (K3),
scores them with the plan evaluator (K1), and performs the round bookkeeping, BPTT and update
(K5/K6) — see csrc/hps_policy.cu. The host only orchestrates launches.

Feature encoding (log1p + z-score of three scalars per layer, ls/policy/features.py:57-130) and
the uniform parameter initialisation (ls/policy/network.py:111-129) run once per training run on
the host with numpy, exactly as the reference does; they are input preparation, not the loop.
With several ranks (torch.distributed), every rank samples the full round, scores its slice of
the G plans, and one all_gather of (cost, status) precedes an identical update on every rank.
"""

from __future__ import annotations

import ctypes as C
import json
import math
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable

import numpy as np

from . import _abi
from .errors import ConfigError, InvariantError, NumericError
from .model import ProvisionerConfig, ScoredPlan, SchedulingPlan

CELL_LSTM = "lstm"
CELL_ELMAN = "elman"
CHECKPOINT_VERSION = 1
UPDATE_NORM_CAP = 50.0          # ls/policy/training.py:41
PENALTY_ADVANTAGE_FACTOR = 10.0  # ls/policy/training.py:47


# ----------------------------------------------------------------------------- features

def _comm_time(layer) -> float:
    vals = [layer.per_type_odt[t] for t in sorted(layer.per_type_odt)]
    return sum(vals) / len(vals) if vals else 0.0


@dataclass(frozen=True)
class LayerFeatures:
    index_onehot: np.ndarray
    kind_onehot: np.ndarray
    input_size_norm: float
    weight_size_norm: float
    comm_time_norm: float

    def as_vector(self) -> np.ndarray:
        tail = np.array([self.input_size_norm, self.weight_size_norm, self.comm_time_norm])
        return np.concatenate([self.index_onehot, self.kind_onehot, tail])


@dataclass(frozen=True)
class FeatureNormalizer:
    """Kind vocabulary + log1p/z-score statistics (ls/policy/features.py:48-90)."""

    max_layers: int
    kinds: tuple
    means: tuple
    stds: tuple

    @classmethod
    def fit(cls, graph, catalog=None, max_layers: int = 64) -> "FeatureNormalizer":
        if catalog is not None and catalog.layer_kinds:
            kinds = tuple(catalog.layer_kinds)
        else:
            kinds = tuple(sorted({l.layer_kind for l in graph.layers}))
        raw = np.array([[math.log1p(l.input_size), math.log1p(l.weight_size),
                         math.log1p(_comm_time(l))] for l in graph.layers])
        return cls(max_layers=max_layers, kinds=kinds,
                   means=tuple(float(x) for x in raw.mean(axis=0)),
                   stds=tuple(float(x) for x in raw.std(axis=0)))

    def zscore(self, slot: int, raw: float) -> float:
        if self.stds[slot] == 0:
            return 0.0
        return (math.log1p(raw) - self.means[slot]) / self.stds[slot]

    @property
    def feature_dim(self) -> int:
        return self.max_layers + len(self.kinds) + 3


def encode_features(graph, catalog, normalizer: FeatureNormalizer) -> list:
    if graph.num_layers > normalizer.max_layers:
        raise ConfigError(f"model '{graph.name}' has {graph.num_layers} layers but the index "
                          f"encoding is {normalizer.max_layers} wide")
    where = {k: i for i, k in enumerate(normalizer.kinds)}
    out = []
    for l in graph.layers:
        if l.layer_kind not in where:
            raise ConfigError(f"layer {l.index} has kind '{l.layer_kind}' not in the declared "
                              f"vocabulary {list(normalizer.kinds)}")
        idx = np.zeros(normalizer.max_layers)
        idx[l.index] = 1.0
        kind = np.zeros(len(normalizer.kinds))
        kind[where[l.layer_kind]] = 1.0
        out.append(LayerFeatures(idx, kind, normalizer.zscore(0, l.input_size),
                                 normalizer.zscore(1, l.weight_size),
                                 normalizer.zscore(2, _comm_time(l))))
    return out


def features_matrix(features: list) -> np.ndarray:
    return np.stack([f.as_vector() for f in features])


# ----------------------------------------------------------------------------- parameters

@dataclass
class PolicyParams:
    cell: str
    w_cell: np.ndarray
    b_cell: np.ndarray
    w_out: np.ndarray
    b_out: np.ndarray
    hidden_size: int

    def __post_init__(self):
        if self.cell not in (CELL_LSTM, CELL_ELMAN):
            raise InvariantError(f"unknown cell kind '{self.cell}'")
        gates = 4 if self.cell == CELL_LSTM else 1
        if self.w_cell.shape[1] != gates * self.hidden_size or self.b_cell.shape != (gates * self.hidden_size,):
            raise InvariantError("cell weight shapes inconsistent with hidden size")
        if self.w_out.shape[0] != self.hidden_size or self.b_out.shape != (self.w_out.shape[1],):
            raise InvariantError("output head shapes inconsistent")

    @property
    def feature_dim(self) -> int:
        return self.w_cell.shape[0] - self.hidden_size

    @property
    def num_types(self) -> int:
        return self.w_out.shape[1]

    def copy(self) -> "PolicyParams":
        return PolicyParams(self.cell, self.w_cell.copy(), self.b_cell.copy(), self.w_out.copy(),
                            self.b_out.copy(), self.hidden_size)

    def flat(self) -> np.ndarray:
        return np.concatenate([a.ravel() for a in (self.w_cell, self.b_cell, self.w_out, self.b_out)])

    def all_finite(self) -> bool:
        return all(np.all(np.isfinite(a)) for a in (self.w_cell, self.b_cell, self.w_out, self.b_out))


def init_params(cell, feature_dim, num_types, hidden_size, init_scale, rng) -> PolicyParams:
    """Uniform(-s, s) in the reference's draw order (ls/policy/network.py:111-129)."""
    gates = 4 if cell == CELL_LSTM else 1
    u = lambda *shape: rng.uniform(-init_scale, init_scale, size=shape)  # noqa: E731
    return PolicyParams(cell=cell, w_cell=u(feature_dim + hidden_size, gates * hidden_size),
                        b_cell=u(gates * hidden_size), w_out=u(hidden_size, num_types),
                        b_out=u(num_types), hidden_size=hidden_size)


# ----------------------------------------------------------------------------- trainer types

@dataclass(frozen=True)
class TrainerConfig:
    rounds: int = 200
    plans_per_round: int = 20
    baseline_rate: float = 0.7
    learning_rate: float = 0.01
    hidden_size: int = 64
    seed: int = 0
    temperature: float = 1.0
    init_scale: float = 0.1
    max_layers: int = 64
    cell: str = CELL_LSTM
    warmup_rounds: int = 0

    def __post_init__(self):
        if not 0.0 < self.baseline_rate <= 1.0:
            raise InvariantError("baseline_rate must be in (0, 1]")
        if self.learning_rate <= 0:
            raise InvariantError("learning_rate must be > 0")
        if self.plans_per_round < 1:
            raise InvariantError("plans_per_round must be >= 1")
        if self.rounds < 0:
            raise InvariantError("rounds must be >= 0")
        if self.warmup_rounds < 0:
            raise InvariantError("warmup_rounds must be >= 0")
        if self.cell not in (CELL_LSTM, CELL_ELMAN):
            raise InvariantError(f"unknown cell kind '{self.cell}'")


@dataclass(frozen=True)
class RoundStats:
    round: int
    mean_cost: float
    best_cost: float
    baseline: float
    entropy: float


@dataclass
class TrainingResult:
    params: PolicyParams
    normalizer: FeatureNormalizer
    history: list = field(default_factory=list)
    best: ScoredPlan | None = None
    round_wall_s: list = field(default_factory=list)  # extension: wall time at each round's end
    sampled_plans: np.ndarray | None = None            # extension: [rounds, G, L] if recorded


def reward(scored) -> float:
    return -scored.cost


def init_policy(graph, catalog, config: TrainerConfig):
    normalizer = FeatureNormalizer.fit(graph, catalog, max_layers=config.max_layers)
    rng = np.random.default_rng([config.seed, 0])
    params = init_params(config.cell, normalizer.feature_dim, catalog.num_types,
                         config.hidden_size, config.init_scale, rng)
    return params, normalizer


# ----------------------------------------------------------------------------- device policy

_DEVICE_COUNTER = (1 << 64) - 1   # hps_policy_sample first_draw: read the device counter


def _lib():
    return _abi.load_library()


def _chk(code, what):
    if code != 0:
        msg = (_lib().hps_policy_last_error() or b"").decode()
        _abi.check(code, f"{what}: {msg}")


class DevicePolicy:
    """Parameters, features and round state of one policy on the current CUDA device."""

    def __init__(self, params: PolicyParams, features: np.ndarray, max_plans: int):
        import torch
        from .instance import _require_cuda
        _require_cuda()
        self.lib = _lib()
        L, D = features.shape
        if D != params.feature_dim:
            raise InvariantError(f"features have dimension {D}, parameters expect {params.feature_dim}")
        self.L, self.D, self.H, self.T = L, D, params.hidden_size, params.num_types
        self.cell = params.cell
        h = C.c_void_p()
        feat = np.ascontiguousarray(features, dtype=np.float64)
        _chk(self.lib.hps_policy_create(L, D, self.H, self.T, 1 if params.cell == CELL_LSTM else 0,
                                        max_plans, feat.ctypes.data_as(C.c_void_p), C.byref(h)),
             "hps_policy_create")
        self.h = h
        self.set_params(params)
        self.device = torch.device("cuda", torch.cuda.current_device())

    def close(self):
        if getattr(self, "h", None):
            self.lib.hps_policy_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_params(self, p: PolicyParams):
        for which, arr in enumerate((p.w_cell, p.b_cell, p.w_out, p.b_out)):
            a = np.ascontiguousarray(arr, dtype=np.float64)
            _chk(self.lib.hps_policy_params(self.h, which, 0, a.ctypes.data_as(C.c_void_p), a.size),
                 "hps_policy_params")

    def get_params(self) -> PolicyParams:
        shapes = [(self.D + self.H, (4 if self.cell == CELL_LSTM else 1) * self.H),
                  ((4 if self.cell == CELL_LSTM else 1) * self.H,), (self.H, self.T), (self.T,)]
        arrs = []
        for which, shp in enumerate(shapes):
            a = np.empty(shp, dtype=np.float64)
            _chk(self.lib.hps_policy_params(self.h, which, 1, a.ctypes.data_as(C.c_void_p), a.size),
                 "hps_policy_params")
            arrs.append(a)
        return PolicyParams(self.cell, arrs[0], arrs[1], arrs[2], arrs[3], self.H)

    def _stream(self):
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def forward(self, temperature: float, probs_out=None):
        _chk(self.lib.hps_policy_forward(self.h, temperature,
                                         C.c_void_p(probs_out.data_ptr()) if probs_out is not None else None,
                                         self._stream()), "hps_policy_forward")

    def sample(self, pcg, first_draw: int, n: int, plans_out):
        _chk(self.lib.hps_policy_sample(self.h, C.byref(pcg), first_draw, n,
                                        C.c_void_p(plans_out.data_ptr()), self._stream()),
             "hps_policy_sample")

    def reinforce(self, cost, status, plans, round_index, temperature, lr, gamma, history,
                  best_plan, best_where):
        _chk(self.lib.hps_policy_reinforce(
            self.h, C.c_void_p(cost.data_ptr()), C.c_void_p(status.data_ptr()),
            C.c_void_p(plans.data_ptr()), plans.shape[0], round_index, temperature, lr, gamma,
            C.c_void_p(history.data_ptr()), C.c_void_p(best_plan.data_ptr()),
            C.c_void_p(best_where.data_ptr()), self._stream()), "hps_policy_reinforce")

    def set_counter(self, round_index: int, draws: int):
        _chk(self.lib.hps_policy_counter(self.h, round_index, draws, self._stream()), "hps_policy_counter")

    def state(self):
        st = (C.c_double * 3)()
        fl = (C.c_int32 * 2)()
        _chk(self.lib.hps_policy_state(self.h, st, fl), "hps_policy_state")
        return tuple(st), tuple(fl)


def policy_forward(params: PolicyParams, features: np.ndarray, temperature: float = 1.0):
    """Device forward; returns (probs [L, T], {}) (the cache stays on the device)."""
    import torch
    if temperature <= 0:
        raise InvariantError("temperature must be > 0 for a forward pass")
    dp = DevicePolicy(params, features, 1)
    probs = torch.empty((features.shape[0], params.num_types), dtype=torch.float64, device=dp.device)
    dp.forward(temperature, probs)
    _, flags = dp.state()
    if flags[0]:
        raise NumericError("non-finite activation in the policy forward pass")
    return probs.cpu().numpy(), {}


def greedy_plan(params: PolicyParams, features: np.ndarray) -> SchedulingPlan:
    probs, _ = policy_forward(params, features, 1.0)
    return SchedulingPlan(tuple(int(np.argmax(row)) for row in probs))


# ----------------------------------------------------------------------------- training

def _dist():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist
    except ImportError:  # pragma: no cover
        pass
    return None


def train(graph, catalog, params0: PolicyParams, config: TrainerConfig, job,
          provisioner_config: ProvisionerConfig = ProvisionerConfig(),
          score_fn: Callable | None = None, group=None,
          record_plans: bool = False, shard: bool = True) -> TrainingResult:
    """REINFORCE training loop (ls/policy/training.py:164-274) with every round on the device.

    ``score_fn`` may be any callable like the reference's; a non-device callable is called on
    the host for each sampled plan (the reference semantics), the default is the device scorer.
    ``shard=False`` keeps the whole round on this rank even when torch.distributed is
    initialised (a round of a few thousand plans is latency-bound: one GPU is faster than a
    per-round all_gather).
    """
    import torch
    from .instance import pcg_from_generator
    from .scoring import PlanScorer, device_instance
    normalizer = FeatureNormalizer.fit(graph, catalog, max_layers=config.max_layers)
    features = features_matrix(encode_features(graph, catalog, normalizer))
    L, T, G = graph.num_layers, catalog.num_types, config.plans_per_round
    dp = DevicePolicy(params0, features, G)
    dev = dp.device
    device_scoring = score_fn is None or isinstance(score_fn, PlanScorer)
    inst = device_instance(graph, catalog, job, provisioner_config) if device_scoring else None
    rng = np.random.default_rng([config.seed, 1])
    pcg = pcg_from_generator(rng)
    dist = _dist() if shard else None
    rank, world = (dist.get_rank(group), dist.get_world_size(group)) if dist else (0, 1)
    lo, hi = G * rank // world, G * (rank + 1) // world
    plans = torch.empty((G, L), dtype=torch.uint8, device=dev)
    cost = torch.empty(G, dtype=torch.float64, device=dev)
    status = torch.empty(G, dtype=torch.uint8, device=dev)
    history = torch.zeros((max(config.rounds, 1), 4), dtype=torch.float64, device=dev)
    best_plan = torch.zeros(L, dtype=torch.uint8, device=dev)
    best_where = torch.full((2,), -1, dtype=torch.int64, device=dev)
    recorded = torch.empty((config.rounds, G, L), dtype=torch.uint8, device=dev) if record_plans else None
    draws = 0      # 64-bit draws consumed by Generator.random() so far
    halves = 0     # 32-bit halves consumed by Generator.integers() (warm-up rounds)
    # HPS_RL_GRAPH=1: on-policy rounds (device scorer, one rank) are captured once as a CUDA
    # graph and replayed; the round number and the PCG64 draw offset live in the policy's device
    # counter, so every replay is the next round. Off by default: a round is device-bound
    # (1.16 ms replayed vs 1.19 ms eager on cfg4) and the capture costs ~17 ms up front, which
    # time-to-best pays (tools/rl_rounds.py; profiles/r2_rl_rounds.log).
    use_graph = (device_scoring and world == 1 and config.rounds > config.warmup_rounds
                 and os.environ.get("HPS_RL_GRAPH", "0") == "1")
    cuda_graph = None

    def on_policy_round():   # forward, sample, score, REINFORCE: stream-ordered, no host sync
        dp.forward(config.temperature)
        dp.sample(pcg, _DEVICE_COUNTER, G, plans)
        out = inst.score(plans, want_k=False)
        cost.copy_(out["cost"])
        status.copy_(out["status"])
        dp.reinforce(cost, status, plans, 0, config.temperature, config.learning_rate,
                     config.baseline_rate, history, best_plan, best_where)

    # round_wall_s[r-1]: seconds from the start of round 1 to the END of round r on the device
    # timeline (CUDA events on the launching stream, read after the final synchronize)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    round_events = []
    for r in range(1, config.rounds + 1):
        if use_graph and r > config.warmup_rounds:
            if cuda_graph is None:
                dp.set_counter(r, draws)
                inst.score(plans, want_k=False)   # first-call setup outside the capture
                torch.cuda.current_stream().synchronize()
                cuda_graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(cuda_graph):
                    on_policy_round()
            cuda_graph.replay()
            draws += G * L
            if recorded is not None:
                recorded[r - 1].copy_(plans)
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            round_events.append(ev)
            if r % 16 == 0 or r == config.rounds:
                torch.cuda.current_stream().synchronize()
            continue
        dp.forward(config.temperature)
        if r <= config.warmup_rounds:
            if T & (T - 1):
                raise ConfigError("warm-up rounds on the device need a power-of-two type count")
            if inst is None:
                inst = device_instance(graph, catalog, job, provisioner_config)
            plans.copy_(inst.random_plans(pcg, halves // L, G))
            halves += G * L
            draws = (halves + 1) // 2
        else:
            dp.sample(pcg, draws, G, plans)
            draws += G * L
        if device_scoring:
            out = inst.score(plans[lo:hi], want_k=False)
            cost[lo:hi].copy_(out["cost"])
            status[lo:hi].copy_(out["status"])
        else:
            host_plans = plans[lo:hi].cpu().numpy()
            sc = [score_fn(SchedulingPlan(tuple(int(x) for x in p))) for p in host_plans]
            cost[lo:hi].copy_(torch.tensor([s.cost for s in sc], dtype=torch.float64))
            status[lo:hi].copy_(torch.tensor([0 if s.feasible else 5 for s in sc], dtype=torch.uint8))
        if world > 1:  # the round's one exchange: everybody's (cost, status) slices
            parts_c = [torch.empty(G * (q + 1) // world - G * q // world, dtype=torch.float64, device=dev)
                       for q in range(world)]
            parts_s = [torch.empty_like(p, dtype=torch.uint8) for p in parts_c]
            dist.all_gather(parts_c, cost[lo:hi].contiguous(), group=group)
            dist.all_gather(parts_s, status[lo:hi].contiguous(), group=group)
            cost.copy_(torch.cat(parts_c))
            status.copy_(torch.cat(parts_s))
        if recorded is not None:
            recorded[r - 1].copy_(plans)
        dp.reinforce(cost, status, plans, r, config.temperature, config.learning_rate,
                     config.baseline_rate, history, best_plan, best_where)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        round_events.append(ev)
        if r % 16 == 0 or r == config.rounds:
            torch.cuda.current_stream().synchronize()
    torch.cuda.synchronize()
    walls = [ev0.elapsed_time(ev) * 1e-3 for ev in round_events]
    _, flags = dp.state()
    if flags[0]:
        raise NumericError("non-finite activation in the policy forward pass")
    if flags[1]:
        raise NumericError("parameters diverged")
    params = dp.get_params()
    res = TrainingResult(params=params, normalizer=normalizer, round_wall_s=walls)
    if recorded is not None:
        res.sampled_plans = recorded.cpu().numpy()
    h = history.cpu().numpy()
    for r in range(config.rounds):
        res.history.append(RoundStats(round=r + 1, mean_cost=float(h[r, 0]), best_cost=float(h[r, 1]),
                                      baseline=float(h[r, 2]), entropy=float(h[r, 3])))
    if config.rounds > 0:
        bp = tuple(int(x) for x in best_plan.cpu().tolist())
        scorer = score_fn if score_fn is not None else PlanScorer(graph, catalog, job, provisioner_config)
        res.best = scorer(SchedulingPlan(bp))
    return res


def save_checkpoint(path, params: PolicyParams, normalizer: FeatureNormalizer, config: TrainerConfig) -> None:
    """Versioned JSON checkpoint, same schema as ls/policy/training.py:277-313."""
    payload = {"version": CHECKPOINT_VERSION,
               "params": {"cell": params.cell, "hidden_size": params.hidden_size,
                          "w_cell": params.w_cell.tolist(), "b_cell": params.b_cell.tolist(),
                          "w_out": params.w_out.tolist(), "b_out": params.b_out.tolist()},
               "normalizer": {"max_layers": normalizer.max_layers, "kinds": list(normalizer.kinds),
                              "means": list(normalizer.means), "stds": list(normalizer.stds)},
               "config": {k: getattr(config, k) for k in ("rounds", "plans_per_round", "baseline_rate",
                                                          "learning_rate", "hidden_size", "seed",
                                                          "temperature", "init_scale", "max_layers",
                                                          "cell")}}
    Path(path).write_text(json.dumps(payload, indent=2) + "\n")


def load_checkpoint(path):
    payload = json.loads(Path(path).read_text())
    if payload.get("version") != CHECKPOINT_VERSION:
        raise InvariantError(f"unsupported checkpoint version {payload.get('version')!r}")
    p = payload["params"]
    params = PolicyParams(p["cell"], np.array(p["w_cell"], dtype=float), np.array(p["b_cell"], dtype=float),
                          np.array(p["w_out"], dtype=float), np.array(p["b_out"], dtype=float),
                          int(p["hidden_size"]))
    n = payload["normalizer"]
    normalizer = FeatureNormalizer(int(n["max_layers"]), tuple(n["kinds"]), tuple(n["means"]),
                                   tuple(n["stds"]))
    return params, normalizer, TrainerConfig(**payload["config"])
