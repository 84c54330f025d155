"""Device-resident scheduling instance: the one object that owns libhps state.

``DeviceInstance`` stages a (graph, catalog, job, provisioner config) instance on the current
CUDA device through ``hps_instance_create`` and exposes the batched entry points of
include/hps.h on torch tensors (torch is plumbing here: device memory and streams).
No method computes anything on the host; without a GPU the constructor raises.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from .errors import ConfigError, NativeUnavailableError
from .model import ProvisionerConfig

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


def _require_cuda():
    if torch is None or not torch.cuda.is_available():
        raise NativeUnavailableError("no CUDA device visible: the plan evaluator has no CPU path")


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def argmin_from_bytes(buf: bytes) -> dict:
    a = _abi.HpsArgmin.from_buffer_copy(buf)
    return {"cost": a.cost, "rank": (a.rank_hi << 64) | a.rank_lo, "evaluated": a.evaluated,
            "feasible": a.feasible, "status": a.status, "flags": a.flags}


class DeviceInstance:
    """Immutable device tables of one instance (stage table, stage-0 exits, ET table)."""

    def __init__(self, graph, catalog, job, config: ProvisionerConfig | None = None,
                 with_ps: bool = True, device=None):
        _require_cuda()
        self.lib = _abi.load_library()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.graph, self.catalog, self.job = graph, catalog, job
        self.config = config if config is not None else ProvisionerConfig()
        self.staged = _abi.StagedDesc(graph, catalog, job, self.config, with_ps)
        self.L, self.T = self.staged.num_layers, self.staged.num_types
        handle = C.c_void_p()
        with torch.cuda.device(self.device):
            _abi.check(self.lib.hps_instance_create(self.staged.ptr, C.byref(handle)),
                       "hps_instance_create")
        self.handle = handle

    def close(self):
        if getattr(self, "handle", None):
            self.lib.hps_instance_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- stage table (build_stages aggregates, ls/domain.py:275-328) ----
    def stage_aggregates(self, type_id: int, first: int, last: int):
        out = (C.c_double * 4)()
        _abi.check(self.lib.hps_stage_table(self.handle, type_id, first, last, out),
                   "hps_stage_table")
        return tuple(out)

    # ---- K1: batched PlanScorer ----
    def score(self, plans, want_k: bool = True, stream=None, mode: str = "optimal",
              cpu_per_gpu: int = 6) -> dict:
        """Score plans (uint8 [n, L] tensor on this device). Returns device tensors.

        ``mode`` 'staratio' / 'stapsratio' runs the static provisioning baselines
        (ls/provisioner.py:516-561) instead of optimize_k1 + add_ps_cores."""
        if plans.dtype != torch.uint8 or plans.dim() != 2 or plans.shape[1] != self.L:
            raise ConfigError(f"plans must be uint8 [n, {self.L}]")
        plans = plans.to(self.device).contiguous()
        n = plans.shape[0]
        dev = self.device
        out = {"cost": torch.empty(n, dtype=torch.float64, device=dev),
               "status": torch.empty(n, dtype=torch.uint8, device=dev),
               "gap": torch.empty(n, dtype=torch.float64, device=dev),
               "ps": torch.empty(n, dtype=torch.int32, device=dev),
               "num_stages": torch.empty(n, dtype=torch.int32, device=dev),
               "k": torch.empty((n, self.L), dtype=torch.int32, device=dev) if want_k else None}
        res = _abi.HpsPlanResults(*(out[k].data_ptr() if out[k] is not None else None
                                    for k in ("cost", "status", "gap", "ps", "num_stages", "k")))
        with torch.cuda.device(dev):
            if mode == "optimal":
                _abi.check(self.lib.hps_score_plans(self.handle, _ptr(plans), n, C.byref(res),
                                                    _stream(stream)), "hps_score_plans")
            else:
                if mode not in _abi.MODE_CODES:
                    raise ConfigError(f"unknown provisioning mode '{mode}'")
                _abi.check(self.lib.hps_score_plans_static(
                    self.handle, _ptr(plans), n, _abi.MODE_CODES[mode], int(cpu_per_gpu),
                    C.byref(res), _stream(stream)), "hps_score_plans_static")
        return out

    # ---- K2: fused enumeration / random sweep argmin ----
    def _argmin_buffer(self):
        return torch.empty(_abi.ARGMIN_NBYTES, dtype=torch.uint8, device=self.device)

    def enum_argmin_async(self, begin: int, end: int, feasible_only: bool = True, stream=None):
        buf = self._argmin_buffer()
        with torch.cuda.device(self.device):
            _abi.check(self.lib.hps_enum_argmin(self.handle, begin, end, 1 if feasible_only else 0,
                                                _ptr(buf), _stream(stream)), "hps_enum_argmin")
        return buf

    def enum_argmin_strided_async(self, first: int, stride: int, count: int,
                                  feasible_only: bool = True, stream=None):
        buf = self._argmin_buffer()
        with torch.cuda.device(self.device):
            _abi.check(self.lib.hps_enum_argmin_strided(self.handle, first, stride, count,
                                                        1 if feasible_only else 0, _ptr(buf),
                                                        _stream(stream)),
                       "hps_enum_argmin_strided")
        return buf

    def enum_argmin_pruned(self, depth: int | None = None, incumbent: float = float("inf"),
                           stream=None):
        """Feasible-only argmin over all T^L plans with certified subtree pruning
        (hps_enum_argmin_pruned): same winner as enum_argmin_async(0, T^L). Returns
        (key, stats) on the host (the call synchronises the stream)."""
        depth = self.default_prune_depth() if depth is None else int(depth)
        buf = self._argmin_buffer()
        stats = _abi.HpsPruneStats()
        with torch.cuda.device(self.device):
            _abi.check(self.lib.hps_enum_argmin_pruned(self.handle, depth, float(incumbent), _ptr(buf),
                                                       C.byref(stats), _stream(stream)),
                       "hps_enum_argmin_pruned")
        st = {f: getattr(stats, f) for f, _ in _abi.HpsPruneStats._fields_ if f != "pad"}
        return self.read_argmin(buf), st

    def default_prune_depth(self) -> int:
        """Prefix depth of the pruned sweep: about 2^16 index ranges, at least T^4 plans each."""
        d = 1
        while d + 1 < self.L and self.T ** (d + 1) <= (1 << 16) and self.T ** (self.L - d - 1) >= self.T ** 4:
            d += 1
        return d

    def plans_argmin_async(self, plans, feasible_only: bool = False, stream=None):
        plans = plans.to(self.device).contiguous()
        buf = self._argmin_buffer()
        with torch.cuda.device(self.device):
            _abi.check(self.lib.hps_plans_argmin(self.handle, _ptr(plans), plans.shape[0],
                                                 1 if feasible_only else 0, _ptr(buf),
                                                 _stream(stream)), "hps_plans_argmin")
        return buf

    def random_argmin_async(self, pcg: "_abi.HpsPcg64", first: int, n: int, stream=None):
        buf = self._argmin_buffer()
        with torch.cuda.device(self.device):
            _abi.check(self.lib.hps_random_argmin(self.handle, C.byref(pcg), first, n, _ptr(buf),
                                                  _stream(stream)), "hps_random_argmin")
        return buf

    def random_plans(self, pcg: "_abi.HpsPcg64", first: int, n: int, stream=None):
        out = torch.empty((n, self.L), dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            _abi.check(self.lib.hps_random_plans(self.handle, C.byref(pcg), first, n, _ptr(out),
                                                 _stream(stream)), "hps_random_plans")
        return out

    def explain(self, plans, status, k=None, stream=None) -> list:
        """InfeasibleError details of scored plans (hps_explain), as HpsExplain records."""
        plans = plans.to(self.device).contiguous()
        n = plans.shape[0]
        out = torch.empty(n * _abi.EXPLAIN_NBYTES, dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            _abi.check(self.lib.hps_explain(self.handle, _ptr(plans), _ptr(status.contiguous()),
                                            _ptr(k.contiguous()) if k is not None else None, n,
                                            _ptr(out), _stream(stream)), "hps_explain")
        raw = bytes(out.cpu().numpy().tobytes())
        m = _abi.EXPLAIN_NBYTES
        return [_abi.HpsExplain.from_buffer_copy(raw[i * m:(i + 1) * m]) for i in range(n)]

    @staticmethod
    def read_argmin(buf) -> dict:
        return argmin_from_bytes(bytes(buf.cpu().numpy().tobytes()))

    # ---- evaluate() (ls/costmodel.py:102-167) for given counts ----
    def report(self, plans, k, ps, stream=None) -> dict:
        plans = plans.to(self.device).contiguous()
        k = k.to(self.device, torch.int32).contiguous()
        ps = ps.to(self.device, torch.int32).contiguous()
        n, dev = plans.shape[0], self.device
        f64 = dict(dtype=torch.float64, device=dev)
        out = {name: torch.zeros((n, self.L), **f64) for name in ("ct", "dt", "et", "tp")}
        out.update(pipeline_tp=torch.empty(n, **f64), exec_time=torch.empty(n, **f64),
                   cost=torch.empty(n, **f64),
                   feasible=torch.empty(n, dtype=torch.uint8, device=dev))
        with torch.cuda.device(dev):
            _abi.check(self.lib.hps_report(
                self.handle, _ptr(plans), _ptr(k), _ptr(ps), n, _ptr(out["ct"]), _ptr(out["dt"]),
                _ptr(out["et"]), _ptr(out["tp"]), _ptr(out["pipeline_tp"]), _ptr(out["exec_time"]),
                _ptr(out["cost"]), _ptr(out["feasible"]), _stream(stream)), "hps_report")
        return out


def pcg_from_generator(rng: np.random.Generator) -> "_abi.HpsPcg64":
    return _abi.pcg64_words(rng.bit_generator.state)
