"""Time hps_score_plans (every plan's outputs) on 2^20 cfg5 random plans, twice (not a bench)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
from paper_2111_10635_b200 import load_fixture
from paper_2111_10635_b200.instance import DeviceInstance, pcg_from_generator
from paper_2111_10635_b200.model import JobParams
g, c, lim = load_fixture("cfg5")
inst = DeviceInstance(g, c, JobParams(lim))
pcg = pcg_from_generator(np.random.default_rng(0))
n = 1 << 20
plans = inst.random_plans(pcg, 0, n)
inst.score(plans[:4096])
for r in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = inst.score(plans)
    e1.record()
    torch.cuda.synchronize()
    print(f"cfg5 batch {n}: {e0.elapsed_time(e1):.1f} ms -> {n / e0.elapsed_time(e1) * 1e3:.3e} plans/s", flush=True)
