"""Run a sweep with the instrumented library (libhps_stats.so) and print the device counters."""
import argparse
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
NAMES = ["plans", "chunks", "chunks_eval", "cands_eval", "probes_exact", "probes_closed", "cert", "cert_fail",
         "tab", "pending", "stages", "unpinned", "ncand", "plans_fast", "cyc_a", "cyc_b", "cyc_c", "cyc_p1",
         "cyc_p2", "n2_restricted", "n2_uncertified", "ideal_survivors", "ideal2_survivors", "near_1e-3"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instance", default="cfg3")
    ap.add_argument("--begin", type=int, default=3 ** 16 // 2)
    ap.add_argument("--count", type=int, default=1 << 16)
    ap.add_argument("--lib", default="libhps_stats.so")
    a = ap.parse_args()
    os.environ["HPS_LIBRARY"] = str(ROOT / "paper_2111_10635_b200" / a.lib)
    import torch
    from paper_2111_10635_b200 import _abi, load_fixture
    from paper_2111_10635_b200.instance import DeviceInstance
    from paper_2111_10635_b200.model import JobParams
    lib = _abi.load_library()
    lib.hps_stats_read.argtypes = [C.c_void_p, C.c_int, C.c_int]
    g, c, limit = load_fixture(a.instance)
    inst = DeviceInstance(g, c, JobParams(limit))
    buf = (C.c_ulonglong * 24)()
    lib.hps_stats_read(buf, 24, 1)
    key = inst.read_argmin(inst.enum_argmin_async(a.begin, a.begin + a.count, True))
    torch.cuda.synchronize()
    lib.hps_stats_read(buf, 24, 0)
    st = dict(zip(NAMES, list(buf)[:len(NAMES)]))
    print(key)
    print(st)
    pf = max(1, int(os.environ.get("STATS_PLANS", "0")) or st["plans_fast"] or 1)
    print({k: round(v / pf, 2) for k, v in st.items()})


if __name__ == "__main__":
    main()
