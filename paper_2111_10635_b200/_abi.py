"""ctypes mirror of include/hps.h and the loader of the in-tree CUDA library.

There is deliberately no CPU path: if ``libhps.so`` is missing, or the process has no
CUDA device, every product entry point raises :class:`NativeUnavailableError`.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import (ConfigError, InvariantError, NativeUnavailableError, NumericError,
                     PlanValidationError, SchedulerError)

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libhps.so"

# per-plan status byte (include/hps.h HPS_ST_*)
ST_OK, ST_MIN_K1, ST_SERIAL, ST_QUOTA_TAU_HI, ST_FLOOR_TAU_HI = 0, 1, 2, 3, 4
ST_NO_CANDIDATE, ST_PS_QUOTA, ST_DEFENSIVE, ST_NO_CPU_TYPE, ST_INVALID = 5, 6, 7, 8, 9
ST_STATIC_NONE = 10
ST_OVERFLOW_FLAG = 0x80
ST_CODE_MASK = 0x7F
STATUS_NAMES = {ST_OK: "ok", ST_MIN_K1: "min_k1", ST_SERIAL: "serial",
                ST_QUOTA_TAU_HI: "quota_at_tau_hi", ST_FLOOR_TAU_HI: "floor_at_tau_hi",
                ST_NO_CANDIDATE: "no_candidate", ST_PS_QUOTA: "ps_quota",
                ST_DEFENSIVE: "defensive", ST_NO_CPU_TYPE: "no_cpu_type", ST_INVALID: "invalid",
                ST_STATIC_NONE: "static_none"}
MODE_CODES = {"staratio": 1, "stapsratio": 2}   # HPS_MODE_* (include/hps.h)

HPS_OK, HPS_E_INVALID_ARG, HPS_E_PLAN, HPS_E_CONFIG, HPS_E_CUDA = 0, 1, 2, 3, 4
HPS_E_NO_CPU_TYPE, HPS_E_NUMERIC = 5, 6
MAX_LAYERS, MAX_TYPES = 64, 16

_dp, _i64p, _u8p = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_uint8)


class HpsInstanceDesc(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_types", C.c_int32),
                ("oct", _dp), ("odt", _dp), ("alpha", _dp), ("beta", _dp),
                ("price_per_hour", _dp), ("quota", _i64p), ("is_cpu", _u8p),
                ("total_samples", C.c_int64), ("epochs", C.c_int64),
                ("batch_size", C.c_int64), ("profile_batch_size", C.c_int64),
                ("throughput_limit", C.c_double), ("ps_cores_per_gpu", C.c_double),
                ("newton_max_iters", C.c_int32), ("newton_tol", C.c_double),
                ("fd_step", C.c_double), ("with_ps", C.c_int32)]


class HpsPlanResults(C.Structure):
    _fields_ = [("cost", C.c_void_p), ("status", C.c_void_p), ("gap", C.c_void_p),
                ("ps", C.c_void_p), ("num_stages", C.c_void_p), ("k", C.c_void_p)]


class HpsArgmin(C.Structure):
    _fields_ = [("cost", C.c_double), ("rank_hi", C.c_uint64), ("rank_lo", C.c_uint64),
                ("evaluated", C.c_uint64), ("feasible", C.c_uint64),
                ("status", C.c_uint32), ("flags", C.c_uint32)]


class HpsPcg64(C.Structure):
    _fields_ = [("state_hi", C.c_uint64), ("state_lo", C.c_uint64),
                ("inc_hi", C.c_uint64), ("inc_lo", C.c_uint64)]


class HpsExplain(C.Structure):
    _fields_ = [("status", C.c_int32), ("stage", C.c_int32), ("side", C.c_int32),
                ("serial_side", C.c_int32), ("type", C.c_int32), ("pad", C.c_int32),
                ("units_hi", C.c_uint64), ("units_lo", C.c_uint64), ("ps", C.c_int64),
                ("serial", C.c_double), ("tau_hi", C.c_double)]


class HpsPruneStats(C.Structure):
    _fields_ = [("prefixes", C.c_uint64), ("survivors", C.c_uint64), ("evaluated", C.c_uint64),
                ("subtree", C.c_uint64), ("incumbent_cost", C.c_double), ("min_bound", C.c_double),
                ("depth", C.c_int32), ("pad", C.c_int32)]


ARGMIN_NBYTES = C.sizeof(HpsArgmin)  # 48
EXPLAIN_NBYTES = C.sizeof(HpsExplain)  # 64


class StagedDesc:
    """An HpsInstanceDesc plus the numpy arrays it points into (kept alive together)."""

    def __init__(self, graph, catalog, job, config, with_ps: bool = True):
        L, T = graph.num_layers, catalog.num_types
        if not 1 <= L <= MAX_LAYERS:
            raise ConfigError(f"{L} layers: the device evaluator supports 1..{MAX_LAYERS}")
        if not 1 <= T <= MAX_TYPES:
            raise ConfigError(f"{T} types: the device evaluator supports 1..{MAX_TYPES}")
        tabs = {}
        for name in ("oct", "odt", "alpha", "beta"):
            arr = np.empty((T, L), dtype=np.float64)
            for l, layer in enumerate(graph.layers):
                table = getattr(layer, "per_type_" + name)
                for t in range(T):
                    # a missing profile entry is a PlanValidationError only for plans that
                    # use it (ls/domain.py:298-305); mark it NaN and let the kernel flag it
                    arr[t, l] = float(table[t]) if t in table else np.nan
            tabs[name] = np.ascontiguousarray(arr)
        self.tabs = tabs
        self.price = np.array([float(t.price_per_hour) for t in catalog.types], dtype=np.float64)
        self.quota = np.array([int(t.quota) for t in catalog.types], dtype=np.int64)
        self.is_cpu = np.array([1 if t.is_cpu else 0 for t in catalog.types], dtype=np.uint8)
        d = HpsInstanceDesc()
        d.num_layers, d.num_types = L, T
        for name in ("oct", "odt", "alpha", "beta"):
            setattr(d, name, tabs[name].ctypes.data_as(_dp))
        d.price_per_hour = self.price.ctypes.data_as(_dp)
        d.quota = self.quota.ctypes.data_as(_i64p)
        d.is_cpu = self.is_cpu.ctypes.data_as(_u8p)
        d.total_samples, d.epochs = int(graph.total_samples), int(graph.epochs)
        d.batch_size, d.profile_batch_size = int(graph.batch_size), int(graph.profile_batch_size)
        d.throughput_limit = float(job.throughput_limit)
        d.ps_cores_per_gpu = float(config.ps_cores_per_gpu)
        d.newton_max_iters = int(config.newton_max_iters)
        d.newton_tol, d.fd_step = float(config.newton_tol), float(config.fd_step)
        d.with_ps = 1 if with_ps else 0
        self.desc = d
        self.num_layers, self.num_types = L, T

    @property
    def ptr(self):
        return C.byref(self.desc)


def pcg64_words(bit_generator_state: dict) -> HpsPcg64:
    """numpy ``Generator.bit_generator.state`` -> HpsPcg64 (has_uint32 must be 0)."""
    st = bit_generator_state["state"]
    if bit_generator_state.get("has_uint32", 0):
        raise InvariantError("generator holds a buffered 32-bit half; start from a fresh state")
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return HpsPcg64(s >> 64, s & m, inc >> 64, inc & m)


_SIGNATURES = {
    "hps_abi_version": (C.c_int, []),
    "hps_error_string": (C.c_char_p, [C.c_int]),
    "hps_last_error": (C.c_char_p, []),
    "hps_instance_create": (C.c_int, [C.POINTER(HpsInstanceDesc), C.POINTER(C.c_void_p)]),
    "hps_instance_destroy": (C.c_int, [C.c_void_p]),
    "hps_stage_table": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, _dp]),
    "hps_score_plans": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64,
                                  C.POINTER(HpsPlanResults), C.c_void_p]),
    "hps_enum_argmin": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int32, C.c_void_p,
                                  C.c_void_p]),
    "hps_plans_argmin": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p,
                                   C.c_void_p]),
    "hps_random_argmin": (C.c_int, [C.c_void_p, C.POINTER(HpsPcg64), C.c_uint64, C.c_uint64,
                                    C.c_void_p, C.c_void_p]),
    "hps_random_plans": (C.c_int, [C.c_void_p, C.POINTER(HpsPcg64), C.c_uint64, C.c_uint64,
                                   C.c_void_p, C.c_void_p]),
    "hps_policy_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                    C.c_int64, C.c_void_p, C.POINTER(C.c_void_p)]),
    "hps_policy_destroy": (C.c_int, [C.c_void_p]),
    "hps_policy_params": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int64]),
    "hps_policy_forward": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]),
    "hps_policy_sample": (C.c_int, [C.c_void_p, C.POINTER(HpsPcg64), C.c_uint64, C.c_int64,
                                    C.c_void_p, C.c_void_p]),
    "hps_policy_reinforce": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                       C.c_int32, C.c_double, C.c_double, C.c_double, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p]),
    "hps_policy_state": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "hps_policy_counter": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]),
    "hps_policy_last_error": (C.c_char_p, []),
    "hps_probe_fp64": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]),
    "hps_stats_read": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    "hps_enum_argmin_strided": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                          C.c_int32, C.c_void_p, C.c_void_p]),
    "hps_launch_count": (C.c_uint64, []),
    "hps_score_plans_static": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                         C.c_void_p, C.c_void_p]),
    "hps_report": (C.c_int, [C.c_void_p] + [C.c_void_p] * 3 + [C.c_int64] + [C.c_void_p] * 9),
    "hps_explain": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                              C.c_void_p, C.c_void_p]),
    "hps_enum_argmin_pruned": (C.c_int, [C.c_void_p, C.c_int32, C.c_double, C.c_void_p,
                                         C.POINTER(HpsPruneStats), C.c_void_p]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None


def load_library(path: Path | None = None):
    """Load libhps.so (built by __graft_entry__.build()); raise loudly when absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("HPS_LIBRARY", LIB_PATH))
    if not p.exists():
        raise NativeUnavailableError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    if lib.hps_abi_version() != 2:
        raise NativeUnavailableError("libhps.so ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def check(code: int, what: str = "") -> None:
    """Map an HPS_E_* return code to the reference's exception classes."""
    if code == HPS_OK:
        return
    lib = load_library()
    msg = (lib.hps_last_error() or b"").decode() or lib.hps_error_string(code).decode()
    text = f"{what}: {msg}" if what else msg
    if code == HPS_E_PLAN:
        raise PlanValidationError(text)
    if code == HPS_E_CONFIG:
        raise ConfigError(text)
    if code in (HPS_E_INVALID_ARG, HPS_E_NO_CPU_TYPE):
        raise InvariantError(text)
    if code == HPS_E_NUMERIC:
        raise NumericError(text)
    if code == HPS_E_CUDA:
        raise NativeUnavailableError(text)
    raise SchedulerError(text)
