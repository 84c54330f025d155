"""Per-kernel summary of an ncu --metrics csv (tools/ncu_ab.sh output): time, warp instructions per
plan, issue activity. usage: ncu_launch_summary.py <csv> [plans]"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    plans = float(sys.argv[2]) if len(sys.argv) > 2 else 4194304.0
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:44]
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[name][r[mi]] += v
        if r[mi] == "gpu__time_duration.sum":
            cnt[name] += 1
    tot = sum(d["gpu__time_duration.sum"] for d in agg.values())
    for k, d in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"])[:8]:
        n = max(cnt[k], 1)
        t = d["gpu__time_duration.sum"]
        print(f"{k:46s} n={cnt[k]:3d} {t / 1e6:8.2f} ms {100 * t / tot:5.1f}%  "
              f"{d['sm__inst_executed.sum'] / plans:8.0f} warp-inst/plan  "
              f"issue {d['smsp__issue_active.avg.pct_of_peak_sustained_active'] / n:5.1f}%")


if __name__ == "__main__":
    main()
