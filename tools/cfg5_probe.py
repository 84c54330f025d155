"""Time the cfg5 random sweep (2^18 plans) and print device stats when the stats build is used."""
import os
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import ctypes as C
import numpy as np
import torch
from paper_2111_10635_b200 import _abi, load_fixture
from paper_2111_10635_b200.instance import DeviceInstance, pcg_from_generator
from paper_2111_10635_b200.model import JobParams
g, c, lim = load_fixture("cfg5")
inst = DeviceInstance(g, c, JobParams(lim))
pcg = pcg_from_generator(np.random.default_rng(0))
n = int(os.environ.get("CFG5_N", 1 << 18))
stats = "stats" in os.environ.get("HPS_LIBRARY", "")
lib = _abi.load_library()
buf = (C.c_ulonglong * 24)()
if stats:
    lib.hps_stats_read(buf, 24, 1)
for r in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    k = inst.read_argmin(inst.random_argmin_async(pcg, 0, n))
    e1.record()
    torch.cuda.synchronize()
    print(f"cfg5 sweep {n}: {e0.elapsed_time(e1):.1f} ms -> {n / e0.elapsed_time(e1) * 1e3:.3e} plans/s", k["cost"])
if stats:
    lib.hps_stats_read(buf, 24, 0)
    names = ["plans", "chunks", "chunks_eval", "cands_eval", "probes_exact", "probes_closed", "cert",
             "cert_fail", "tab", "pending", "stages", "unpinned", "ncand", "plans_fast", "cyc_A", "cyc_B", "cyc_C"]
    st = dict(zip(names, list(buf)))
    pf = max(1, st["plans_fast"])
    print({k: round(v / pf, 2) for k, v in st.items()}, "pending frac", st["pending"] / max(1, st["plans"]))
