"""The one exchange of the sharded sweep (48-byte argmin keys, all_gather + deterministic merge)
on CPU with gloo, world_size 2 — the host-side logic of the multi-GPU path."""
import ctypes
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2111_10635_b200 import _abi
from paper_2111_10635_b200.search import allgather_argmin, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _key_bytes(cost, rank, evaluated, feasible, status=0, flags=0):
    k = _abi.HpsArgmin(cost, rank >> 64, rank & ((1 << 64) - 1), evaluated, feasible, status, flags)
    return torch.frombuffer(bytearray(bytes(k)), dtype=torch.uint8).clone()


def _worker(r, world, port, keys, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=r, world_size=world)
    try:
        kr = keys[r]
        buf = (torch.cat([_key_bytes(*k) for k in kr]) if isinstance(kr, list)
               else _key_bytes(*kr))
        merged = allgather_argmin(buf)
        out_q.put((r, merged))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("keys,expect", [
    ([(0.5, 10, 100, 7), (0.25, 99, 100, 3)], (0.25, 99, 200, 10)),
    ([(0.25, 12, 50, 1), (0.25, 7, 50, 2)], (0.25, 7, 100, 3)),        # cost tie -> smaller rank
    ([(float("inf"), 2 ** 64 - 1, 10, 0), (1.5, 2 ** 100 + 5, 10, 1)], (1.5, 2 ** 100 + 5, 20, 1)),
    # several keys per rank in one buffer
    ([[(0.5, 1, 5, 1), (0.3, 40, 5, 2)], [(0.3, 17, 5, 3), (0.9, 60, 5, 4)]], (0.3, 17, 20, 10)),
])
def test_allgather_argmin_gloo_world2(keys, expect):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, keys, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        m = res[r]
        assert (m["cost"], m["rank"], m["evaluated"], m["feasible"]) == expect


def test_shards_partition_enumeration_for_any_world():
    total = 3 ** 16
    for world in (1, 2, 4, 8):
        spans = [shard_range(0, total, r, world) for r in range(world)]
        assert sum(b - a for a, b in spans) == total
