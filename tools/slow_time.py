"""Time the >4096-breakpoint slow path alone: score the cfg3 plans that overflow (diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_10635_b200 import load_fixture  # noqa: E402
from paper_2111_10635_b200.instance import DeviceInstance  # noqa: E402
from paper_2111_10635_b200.model import JobParams  # noqa: E402

g, c, lim = load_fixture("cfg3")
inst = DeviceInstance(g, c, JobParams(lim))
T, L = 3, 16
idx = np.arange(0, 3 ** 16, 97, dtype=np.int64)[:400000]
digits = np.stack([(idx // 3 ** (L - 1 - l)) % 3 for l in range(L)], 1).astype(np.uint8)
plans = torch.from_numpy(digits).cuda()
out = inst.score(plans)
ovf = ((out["status"] & 0x80) != 0)
sel = plans[ovf]
print("overflow plans in sample:", int(ovf.sum()))
for _ in range(2):
    inst.score(sel)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    inst.score(sel)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"{sel.shape[0]} overflow plans: {ms:.2f} ms -> {ms * 1e3 / max(1, sel.shape[0]):.2f} us/plan")

