"""Reference policy_forward outputs (ls/policy/network.py:147-200) at the initial parameters of
cfg1/cfg4 (seed 0) and cfg5 (seed 3), plus features and init-parameter checksums (test infra)."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent))
import layersched as ls  # noqa: E402
from layersched.policy import training as tr, network as nw, features as ft  # noqa: E402
from make_rl_goldens import load  # noqa: E402

out = []
for name, seed in (("cfg1", 0), ("cfg4", 0), ("cfg5", 3)):
    g, c, job = load(name)
    cfg = tr.TrainerConfig(seed=seed)
    params, norm = tr.init_policy(g, c, cfg)
    X = ft.features_matrix(ft.encode_features(g, c, norm))
    probs, _ = nw.policy_forward(params, X, 1.0)
    out.append({"instance": name, "seed": seed, "features": [[v.hex() for v in row] for row in X],
                "probs": [[v.hex() for v in row] for row in probs],
                "w_cell_sum": float(params.w_cell.sum()).hex(),
                "entropy": nw.entropy_of(probs).hex()})
(Path(__file__).resolve().parent / "rl_probs.json").write_text(json.dumps(out))
print("ok", [o["instance"] for o in out])
