"""Each rank times the SAME enumeration range on its own GPU: separates per-GPU speed
variance from work imbalance between shards (diagnostic)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_10635_b200 import load_fixture  # noqa: E402
from paper_2111_10635_b200.instance import DeviceInstance  # noqa: E402
from paper_2111_10635_b200.model import JobParams  # noqa: E402
from paper_2111_10635_b200.search import shard_range  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", 0))
world = int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(local)
g, c, lim = load_fixture("cfg3")
inst = DeviceInstance(g, c, JobParams(lim))
total = 3 ** 16
res = {}
for label, (lo, hi) in [("same", (0, total // 4))] + [(f"shard{r}", shard_range(0, total, r, 4)) for r in range(4)]:
    for _ in range(2):
        inst.read_argmin(inst.enum_argmin_async(lo, hi, True))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        inst.enum_argmin_async(lo, hi, True)
    e1.record()
    torch.cuda.synchronize()
    res[label] = round(e0.elapsed_time(e1) / 2, 1)
print(local, res, flush=True)
