"""Full-size parity of the device sweeps (through the C-ABI).

* every plan of each exhaustive configuration, cfg3's 43,046,721 included, against the oracle's
  sweep digest (tests/golden/sweep_digests.json, made by tests/golden/make_sweep_digests.py; the
  winners there are re-scored by the reference itself): winner, feasible count, per-status counts
  and a digest over every plan's cost/gap bits, status, PS cores and per-stage counts;
* the literal path (HPS_FORCE_LITERAL) over the same full sweeps gives the same digest;
* the slow path's pending list is sized per super-chunk (HPS_SUPERCHUNK): results do not depend
  on the chunking, and more than 2^20 pending plans in one call are all evaluated.
"""
import json
import os
from contextlib import contextmanager

import numpy as np
import pytest

from goldens import GOLDEN, expected, instance, plans_array, read_jsonl
from sweep_digest import digest_sum, plan_hashes

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DIGESTS = json.loads((GOLDEN / "sweep_digests.json").read_text())


@contextmanager
def env(**kv):
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update({k: str(v) for k, v in kv.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _dev(name, **kv):
    from paper_2111_10635_b200.instance import DeviceInstance
    g, c, job = instance(name)
    with env(**kv):
        return DeviceInstance(g, c, job)


def decode(idx, T, L):
    out = torch.empty((idx.shape[0], L), dtype=torch.uint8, device=idx.device)
    x = idx.clone()
    for l in range(L - 1, -1, -1):
        out[:, l] = (x % T).to(torch.uint8)
        x //= T
    return out


def sweep_digest(inst, total, chunk=1 << 22):
    """(digest, feasible, by_status) of every plan in [0, total) scored through hps_score_plans."""
    dig, feas, by = 0, 0, {}
    for b in range(0, total, chunk):
        idx = torch.arange(b, min(total, b + chunk), dtype=torch.int64, device="cuda")
        out = inst.score(decode(idx, inst.T, inst.L))
        h = plan_hashes(idx, out["cost"], out["status"], out["gap"], out["ps"], out["num_stages"], out["k"])
        dig = (dig + digest_sum(h)) & ((1 << 64) - 1)
        code = (out["status"] & 0x7F).to(torch.int64)
        cnt = torch.bincount(code, minlength=16).cpu().tolist()
        for c, n in enumerate(cnt):
            if n:
                by[str(c)] = by.get(str(c), 0) + n
        feas += cnt[0]
        del out, h
    return dig, feas, by


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "nce5", "quota", "cfg4", "cfg3"])
def test_full_sweep_matches_oracle_digest(name):
    ref = DIGESTS[name]
    inst = _dev(name)
    total = inst.T ** inst.L
    key = inst.read_argmin(inst.enum_argmin_async(0, total, True))
    assert key["rank"] == ref["best_index"] and key["cost"] == float.fromhex(ref["best_cost"])
    assert key["feasible"] == ref["feasible"] and key["evaluated"] == total
    dig, feas, by = sweep_digest(inst, total)
    assert feas == ref["feasible"] and by == ref["by_status"]
    assert str(dig) == ref["digest"], name


@pytest.mark.parametrize("name", ["cfg4", "cfg3"])
def test_literal_path_full_sweep_digest(name):
    ref = DIGESTS[name]
    inst = _dev(name, HPS_FORCE_LITERAL=1)
    total = inst.T ** inst.L
    key = inst.read_argmin(inst.enum_argmin_async(0, total, True))
    assert key["rank"] == ref["best_index"] and key["feasible"] == ref["feasible"]
    dig, _, _ = sweep_digest(inst, total)
    assert str(dig) == ref["digest"]


def test_superchunk_invariance():
    from paper_2111_10635_b200.instance import pcg_from_generator
    big, small = _dev("cfg4"), _dev("cfg4", HPS_SUPERCHUNK=4099)
    total = 2 ** 16
    kb = big.read_argmin(big.enum_argmin_async(0, total, True))
    ks = small.read_argmin(small.enum_argmin_async(0, total, True))
    assert kb == ks and kb["rank"] == 4030
    kb = big.read_argmin(big.enum_argmin_strided_async(3, 7, 9000, True))
    ks = small.read_argmin(small.enum_argmin_strided_async(3, 7, 9000, True))
    assert kb == ks
    assert sweep_digest(big, total) == sweep_digest(small, total)
    b5, s5 = _dev("cfg5"), _dev("cfg5", HPS_SUPERCHUNK=3001)
    pcg = pcg_from_generator(np.random.default_rng(0))
    kb = b5.read_argmin(b5.random_argmin_async(pcg, 1000, 20000))
    ks = s5.read_argmin(s5.random_argmin_async(pcg, 1000, 20000))
    assert kb == ks


def test_pending_list_holds_more_than_2p20_plans():
    """1.2 M copies of the reference's overflow-path plans in one call: every one is evaluated
    (the round-1 list held 2^20 and dropped the rest)."""
    records = [r for r in read_jsonl("ovf.jsonl.gz") if r["instance"] == "tight16"]
    assert records and all(r["ovf"] for r in records)
    reps = (1_200_000 + len(records) - 1) // len(records)
    plans = np.tile(plans_array(records), (reps, 1))
    inst = _dev("tight16")
    out = inst.score(torch.from_numpy(plans).cuda())
    cost, status, _, ps, ovf = expected(records)
    got = out["cost"].cpu().numpy().view(np.int64)
    assert np.array_equal(got, np.tile(cost.view(np.int64), reps))
    assert np.array_equal((out["status"].cpu().numpy() & 0x7F).astype(np.int64), np.tile(status, reps))
    assert np.array_equal(out["ps"].cpu().numpy().astype(np.int64), np.tile(ps, reps))
    # and in an argmin: the minimum over the tiled batch is the minimum over the records
    key = inst.read_argmin(inst.plans_argmin_async(torch.from_numpy(plans).cuda(), False))
    assert key["cost"] == cost.min()


@pytest.mark.parametrize("name,depth", [("cfg3", 10), ("cfg3", 8), ("cfg4", 8), ("cfg2", 4), ("quota", 8),
                                        ("cfg1", 2)])
def test_pruned_sweep_returns_the_full_sweep_winner(name, depth):
    """Certified subtree pruning: same winner (index and cost) as the exhaustive sweep."""
    ref = DIGESTS[name]
    inst = _dev(name)
    key, st = inst.enum_argmin_pruned(depth)
    assert key["rank"] == ref["best_index"] and key["cost"] == float.fromhex(ref["best_cost"]), (key, st)
    assert st["evaluated"] == key["evaluated"] <= inst.T ** inst.L
    assert st["prefixes"] == inst.T ** depth
    # with the optimum as the incumbent every surviving range holds a plan within the bound
    key2, st2 = inst.enum_argmin_pruned(depth, incumbent=float.fromhex(ref["best_cost"]))
    assert key2["rank"] == ref["best_index"] and st2["survivors"] <= st["survivors"] + 1


def test_pruned_brute_force_drop_in():
    from paper_2111_10635_b200.search import brute_force
    g, c, job = instance("cfg4")
    a = brute_force(g, c, job)
    b = brute_force(g, c, job, prune=True)
    assert a.plan == b.plan and a.cost == b.cost and a.evaluations == b.evaluations == 2 ** 16


def test_cfg5_stream_fast_literal_and_oracle():
    """BASELINE cfg5 (64 layers x 4 types): the first 2^20 plans of default_rng(0) (the 1e9 sweep's
    stream) scored by the fast and the literal paths are identical; a strided 1/64 sample equals the
    oracle; the fused random_argmin equals the argmin of the scored outputs."""
    import oracle
    from goldens import staged
    from paper_2111_10635_b200.instance import pcg_from_generator
    n = 1 << 20
    fast, lit = _dev("cfg5"), _dev("cfg5", HPS_FORCE_LITERAL=1)
    pcg = pcg_from_generator(np.random.default_rng(0))
    plans = fast.random_plans(pcg, 0, n)
    a, b = fast.score(plans), lit.score(plans)
    idx = torch.arange(n, dtype=torch.int64, device="cuda")
    ha = plan_hashes(idx, a["cost"], a["status"], a["gap"], a["ps"], a["num_stages"], a["k"])
    hb = plan_hashes(idx, b["cost"], b["status"], b["gap"], b["ps"], b["num_stages"], b["k"])
    assert torch.equal(ha, hb)
    sel = torch.arange(0, n, 64, device="cuda")
    g, c, job = instance("cfg5")
    ref = oracle.score_batch(staged(g, c, job), plans[sel].cpu().numpy())
    assert np.array_equal(a["cost"][sel].cpu().numpy().view(np.int64), ref["cost"].view(np.int64))
    assert np.array_equal(a["status"][sel].cpu().numpy(), ref["status"])
    assert np.array_equal(a["k"][sel].cpu().numpy(), ref["k"])
    key = fast.read_argmin(fast.random_argmin_async(pcg, 0, n))
    cost = a["cost"]
    m = cost.min()
    # penalised plans included (ls/baselines.py:275-278); ties -> lexicographically smaller plan
    ties = torch.nonzero(cost == m)[:, 0].cpu().numpy()
    best = min(ties, key=lambda i: tuple(plans[i].cpu().tolist()))
    assert key["cost"] == float(m) and key["evaluated"] == n
    from paper_2111_10635_b200.search import decode_packed
    assert list(decode_packed(key["rank"], 4, 64)) == plans[best].cpu().tolist()
