"""One enumeration sweep over a sub-range of a fixture (used under ncu; not a bench)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instance", default="cfg3")
    ap.add_argument("--begin", type=int, default=3 ** 16 // 2)
    ap.add_argument("--count", type=int, default=1 << 20)
    ap.add_argument("--repeat", type=int, default=2)
    a = ap.parse_args()
    import torch
    from paper_2111_10635_b200 import load_fixture
    from paper_2111_10635_b200.instance import DeviceInstance
    from paper_2111_10635_b200.model import JobParams
    g, c, limit = load_fixture(a.instance)
    inst = DeviceInstance(g, c, JobParams(limit))
    import time
    for r in range(a.repeat):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        buf = inst.enum_argmin_async(a.begin, a.begin + a.count, True)
        e1.record()
        key = inst.read_argmin(buf)
        print(f"sweep {a.count} plans: {e0.elapsed_time(e1):.2f} ms", flush=True)
    torch.cuda.synchronize()
    print(key)


if __name__ == "__main__":
    main()
