import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
from goldens import instance
from paper_2111_10635_b200 import policy as pol
g, c, job = instance("cfg1")
cfg = pol.TrainerConfig(rounds=3, plans_per_round=64, seed=0)
p0, _ = pol.init_policy(g, c, cfg)
r = pol.train(g, c, p0, cfg, job)
print("ok", os.environ.get("HPS_RL_GRAPH"), [h.baseline for h in r.history])
