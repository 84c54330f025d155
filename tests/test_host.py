"""CPU-only tests: the C-ABI library loads and exports include/hps.h, host-side logic
(sharding, key merge, decoding, RNG replicas, file I/O), and loud failure without a GPU."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import oracle
from goldens import instance, staged
from paper_2111_10635_b200 import _abi, graphio
from paper_2111_10635_b200.errors import NativeUnavailableError
from paper_2111_10635_b200.search import (decode_index, decode_packed, merge_keys, shard_range)

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_header_symbol():
    lib = _abi.load_library()
    header = (ROOT / "include" / "hps.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|const char\*|uint64_t)\s+(hps_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_abi.EXPORTED_SYMBOLS)
    assert lib.hps_abi_version() == 2


def test_abi_struct_sizes_match_header():
    assert ctypes.sizeof(_abi.HpsArgmin) == 48
    assert ctypes.sizeof(_abi.HpsPcg64) == 32
    assert ctypes.sizeof(_abi.HpsPlanResults) == 48


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2111_10635_b200.instance import DeviceInstance
    g, c, job = instance("cfg1")
    with pytest.raises(NativeUnavailableError):
        DeviceInstance(g, c, job)
    from paper_2111_10635_b200.scoring import PlanScorer
    from paper_2111_10635_b200.model import SchedulingPlan
    with pytest.raises(NativeUnavailableError):
        PlanScorer(g, c, job)(SchedulingPlan((0, 0, 1, 1)))


def test_shards_cover_range_exactly():
    for n, w in [(3 ** 16, 8), (7, 3), (1, 8), (65536, 2)]:
        parts = [shard_range(0, n, r, w) for r in range(w)]
        assert parts[0][0] == 0 and parts[-1][1] == n
        assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))


def test_strided_shards_partition_range():
    from paper_2111_10635_b200.search import shard_strided
    for b, n, w in [(0, 3 ** 16, 8), (0, 3 ** 16, 4), (7, 100, 3), (0, 5, 8), (3, 1, 2)]:
        got = []
        for r in range(w):
            first, stride, count = shard_strided(b, b + n, r, w)
            got += [first + j * stride for j in range(min(count, 50000))]
        if n <= 50000:
            assert sorted(got) == list(range(b, b + n))
        else:
            assert sum(shard_strided(b, b + n, r, w)[2] for r in range(w)) == n


def test_merge_keys_is_deterministic_min():
    keys = [{"cost": 2.0, "rank": 5, "evaluated": 10, "feasible": 3, "flags": 0, "status": 0},
            {"cost": 1.0, "rank": 9, "evaluated": 10, "feasible": 4, "flags": 0, "status": 0},
            {"cost": 1.0, "rank": 7, "evaluated": 10, "feasible": 5, "flags": 1, "status": 0}]
    for perm in ([0, 1, 2], [2, 1, 0], [1, 2, 0]):
        m = merge_keys([keys[i] for i in perm])
        assert (m["cost"], m["rank"], m["feasible"], m["flags"]) == (1.0, 7, 12, 1)


def test_decoders_match_itertools_order():
    import itertools
    for T, L in [(2, 4), (3, 5), (4, 3)]:
        for i, a in enumerate(itertools.product(range(T), repeat=L)):
            assert decode_index(i, T, L) == a
    bits = 2
    a = (3, 0, 2, 1)
    rank = sum(d << ((3 - l) * bits) for l, d in enumerate(a))
    assert decode_packed(rank, 4, 4) == a


@pytest.mark.parametrize("T,L", [(2, 16), (3, 16), (4, 64), (3, 5), (1, 4)])
def test_oracle_rng_replica_matches_numpy(T, L):
    pcg = _abi.pcg64_words(np.random.default_rng(11).bit_generator.state)
    got = oracle.random_plans(pcg, T, L, 200)
    rng = np.random.default_rng(11)
    ref = np.stack([rng.integers(0, T, L) for _ in range(200)]).astype(np.uint8)
    assert np.array_equal(got, ref)


def test_graph_io_round_trip(tmp_path):
    g, c, limit = graphio.load_fixture("cfg5")
    graphio.save_model_graph(g, tmp_path / "g.json")
    graphio.save_catalog(c, tmp_path / "c.json")
    assert graphio.load_model_graph(tmp_path / "g.json") == g
    assert graphio.load_catalog(tmp_path / "c.json") == c


def test_builders_reproduce_fixture():
    """resize_model/catalog_with_gpu_variants/simulate_type_variants rebuild cfg5 exactly."""
    g4, c4, _ = graphio.load_fixture("cfg4")
    c = graphio.catalog_with_gpu_variants(c4, 4)
    g = graphio.simulate_type_variants(graphio.resize_model(g4, 64), c)
    gf, cf, _ = graphio.load_fixture("cfg5")
    assert graphio.graph_to_dict(g) == graphio.graph_to_dict(gf)
    assert graphio.catalog_to_dict(c) == graphio.catalog_to_dict(cf)


def test_oracle_brute_force_goldens():
    for name, plan, cost in [("cfg1", (0, 0, 1, 1), 0.028293565538194444),
                             ("cfg2", (0, 0, 0, 0, 0, 1, 1, 1), 0.022149522569444444)]:
        g, c, job = instance(name)
        bc, bi, _ = oracle.enum_argmin(staged(g, c, job), 0, c.num_types ** g.num_layers)
        assert bc == cost
        assert decode_index(bi, c.num_types, g.num_layers) == plan
