"""Order-independent digest of a sweep's per-plan outputs, computed from device tensors.

Same function as the oracle's hpso_plan_hash / hpso_enum_digest (oracle/hps_oracle.c): per plan a
splitmix64 chain over (enumeration index, cost bits, gap bits, status | ps << 8 | S << 40,
k[0..L) with k and ps zeroed unless status == OK); the digest is the wrapping 64-bit sum.
Test infrastructure: used by tests/test_gpu_sweep.py to pin EVERY plan of a full sweep.
"""
from __future__ import annotations

import torch

_M64 = (1 << 64) - 1


def _s(v: int) -> int:  # uint64 constant as the int64 torch stores
    v &= _M64
    return v - (1 << 64) if v >= 1 << 63 else v


C0, C1, C2 = _s(0x9E3779B97F4A7C15), _s(0xBF58476D1CE4E5B9), _s(0x94D049BB133111EB)


def _lsr(x, k: int):
    return (x >> k) & ((1 << (64 - k)) - 1)


def smix(x):
    x = x + C0
    x = (x ^ _lsr(x, 30)) * C1
    x = (x ^ _lsr(x, 27)) * C2
    return x ^ _lsr(x, 31)


def plan_hashes(idx, cost, status, gap, ps, nstages, k):
    """int64 [n] hashes; idx int64 [n], cost/gap float64 [n], status uint8 [n], ps/nstages int32
    [n], k int32 [n, L]."""
    st = status.to(torch.int64)
    ok = (st & 0x7F) == 0
    h = smix(idx.to(torch.int64))
    h = smix(h ^ cost.contiguous().view(torch.int64))
    h = smix(h ^ gap.contiguous().view(torch.int64))
    psz = torch.where(ok, ps.to(torch.int64), torch.zeros_like(st))
    h = smix(h ^ (st | (psz << 8) | (nstages.to(torch.int64) << 40)))
    kk = torch.where(ok[:, None], k.to(torch.int64) & 0xFFFFFFFF, torch.zeros_like(k, dtype=torch.int64))
    for s in range(k.shape[1]):
        h = smix(h ^ kk[:, s] ^ (s << 32))
    return h


def digest_sum(h) -> int:
    """wrapping uint64 sum of int64 hashes (exact: summed in 32-bit halves)."""
    lo = (h & 0xFFFFFFFF).sum().item()
    hi = _lsr(h, 32).sum().item()
    return (lo + (hi << 32)) & _M64
