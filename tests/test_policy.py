"""Policy path: host-side feature/param preparation vs the reference (CPU), and the device
forward / sampler / REINFORCE rounds vs the reference's traces (GPU)."""
import gzip
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from goldens import instance
from paper_2111_10635_b200 import policy as pol

GOLDEN = Path(__file__).resolve().parent / "golden"


def _probs_goldens():
    return json.loads((GOLDEN / "rl_probs.json").read_text())


def _traces():
    with gzip.open(GOLDEN / "rl_traces.json.gz", "rt") as f:
        return json.load(f)


@pytest.mark.parametrize("item", _probs_goldens(), ids=lambda it: it["instance"])
def test_features_and_init_match_reference(item):
    g, c, job = instance(item["instance"])
    cfg = pol.TrainerConfig(seed=item["seed"])
    params, norm = pol.init_policy(g, c, cfg)
    X = pol.features_matrix(pol.encode_features(g, c, norm))
    ref = np.array([[float.fromhex(v) for v in row] for row in item["features"]])
    assert np.array_equal(X, ref)  # bit-exact host preparation
    assert float(params.w_cell.sum()).hex() == item["w_cell_sum"]


@pytest.mark.gpu
@pytest.mark.parametrize("item", _probs_goldens(), ids=lambda it: it["instance"])
def test_device_forward_matches_reference(item):
    g, c, job = instance(item["instance"])
    params, norm = pol.init_policy(g, c, pol.TrainerConfig(seed=item["seed"]))
    X = pol.features_matrix(pol.encode_features(g, c, norm))
    probs, _ = pol.policy_forward(params, X, 1.0)
    ref = np.array([[float.fromhex(v) for v in row] for row in item["probs"]])
    # OpenBLAS vs device dot-product order: ulp-level agreement (SURVEY.md §7 hard part 4)
    assert np.max(np.abs(probs - ref) / ref) < 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("idx", [0, 1, 2, 3])
def test_training_rounds_match_reference(idx):
    tr = _traces()[idx]
    g, c, job = instance(tr["instance"])
    cfg = pol.TrainerConfig(rounds=tr["rounds"], plans_per_round=tr["plans_per_round"], seed=tr["seed"])
    params0, _ = pol.init_policy(g, c, cfg)
    res = pol.train(g, c, params0, cfg, job, record_plans=True)
    for r, (h, st) in enumerate(zip(tr["history"], res.history)):
        digest = hashlib.sha1(res.sampled_plans[r].tobytes()).hexdigest()
        assert digest == h["plans_sha1"], f"round {r + 1}: sampled plans differ"
        assert st.mean_cost.hex() == h["mean_cost"], r
        assert st.best_cost.hex() == h["best_cost"], r
        # baseline/entropy pass through the policy's dot products only via the plans (exact) and
        # the probabilities (ulp-level): require exact baselines, near-exact entropies
        assert st.baseline.hex() == h["baseline"], r
        assert abs(st.entropy - float.fromhex(h["entropy"])) <= 1e-12 * abs(st.entropy)
    assert list(res.best.plan.assignment) == tr["best_plan"]
    assert res.best.cost.hex() == tr["best_cost"]
    final_norm = float(np.linalg.norm(res.params.flat()))
    assert abs(final_norm - float.fromhex(tr["final_params_norm"])) <= 1e-9 * final_norm


@pytest.mark.gpu
def test_graph_replayed_rounds_equal_eager_rounds(monkeypatch):
    """The CUDA-graph round (device round counter) and the eager round run the same kernels."""
    g, c, job = instance("cfg1")
    cfg = pol.TrainerConfig(rounds=40, plans_per_round=64, seed=1)
    params0, _ = pol.init_policy(g, c, cfg)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("HPS_RL_GRAPH", mode)   # eager / CUDA-graph replay
        out[mode] = pol.train(g, c, params0, cfg, job, record_plans=True)
    a, b = out["0"], out["1"]
    assert np.array_equal(a.sampled_plans, b.sampled_plans)
    assert [h.baseline.hex() for h in a.history] == [h.baseline.hex() for h in b.history]
    assert np.array_equal(a.params.flat(), b.params.flat())


CFG4_FULL = GOLDEN / "rl_traces_cfg4_200.json.gz"


@pytest.mark.gpu
@pytest.mark.skipif(not CFG4_FULL.exists(), reason="cfg4 200-round golden not generated")
def test_cfg4_all_200_rounds_match_reference():
    """BASELINE cfg4 (CTRDNN16, 4096 plans x 200 rounds): every round's sampled plans, costs and
    baseline equal the reference trainer's (tests/golden/make_rl_goldens.py --cfg4-full)."""
    with gzip.open(CFG4_FULL, "rt") as f:
        tr = json.load(f)
    g, c, job = instance(tr["instance"])
    cfg = pol.TrainerConfig(rounds=tr["rounds"], plans_per_round=tr["plans_per_round"], seed=tr["seed"])
    params0, _ = pol.init_policy(g, c, cfg)
    res = pol.train(g, c, params0, cfg, job, record_plans=True)
    for r, (h, st) in enumerate(zip(tr["history"], res.history)):
        assert hashlib.sha1(res.sampled_plans[r].tobytes()).hexdigest() == h["plans_sha1"], r + 1
        assert st.mean_cost.hex() == h["mean_cost"] and st.best_cost.hex() == h["best_cost"], r + 1
        assert st.baseline.hex() == h["baseline"], r + 1
        assert abs(st.entropy - float.fromhex(h["entropy"])) <= 1e-12 * abs(st.entropy)
    assert list(res.best.plan.assignment) == tr["best_plan"]
    final_norm = float(np.linalg.norm(res.params.flat()))
    assert abs(final_norm - float.fromhex(tr["final_params_norm"])) <= 1e-9 * final_norm
