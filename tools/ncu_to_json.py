"""Condense an ncu --metrics launch list of `bench.py` into the JSON files bench.py reports from
(profiles/r2_launches_bench_summary.json, profiles/r2_ncu_metrics.json).

usage: ncu_to_json.py <launches.csv> <plans swept under ncu> <out_prefix>

Per kernel: launches, summed duration and share of the listed GPU time, DRAM bytes per plan, warp
instructions per plan, and the launch-averaged issue activity, active threads per warp
instruction and FP64-pipe activity. ncu times are cold-cache and serialised: shares, not
absolute times, are what compare with the bench.
"""
import collections
import csv
import json
import sys

METRICS = {
    "gpu__time_duration.sum": "ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__inst_executed.sum": "inst",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_warp_inst",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
}
AVERAGED = {"issue_active_pct", "threads_per_warp_inst", "fp64_pipe_pct"}
SWEEP_KERNELS = ("stage_kernel", "bisect_kernel", "prep_kernel", "candidate_kernel", "slow_kernel",
                 "stage_kernel_h", "bisect_kernel_h", "prep_kernel_h", "candidate_kernel_h", "init_parts_kernel",
                 "finish_argmin", "merge_argmin")


def main():
    path, plans, prefix = sys.argv[1], float(sys.argv[2]), sys.argv[3]
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = collections.defaultdict(dict)   # launch id -> metrics
    names = {}
    for r in rows[1:]:
        if len(r) <= vi or r[mi] not in METRICS:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        per[r[ii]][METRICS[r[mi]]] = v
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "").replace("hps::", "")
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    for lid, m in per.items():
        k = names[lid]
        agg[k]["launches"] += 1
        for f, v in m.items():
            agg[k][f] += v
    sweep = {k: d for k, d in agg.items() if k.split("<")[0] in SWEEP_KERNELS}
    tot = sum(d["ns"] for d in sweep.values())
    kernels = {}
    for k, d in sorted(sweep.items(), key=lambda x: -x[1]["ns"]):
        n = d["launches"]
        kernels[k] = {"launches": int(n), "ms": d["ns"] / 1e6, "share": d["ns"] / tot,
                      "dram_bytes_per_plan": (d["dram_read"] + d["dram_write"]) / plans,
                      "warp_inst_per_plan": d["inst"] / plans,
                      **{f: d[f] / n for f in AVERAGED if f in d}}
    dram = sum(v["dram_bytes_per_plan"] for v in kernels.values())
    summary = {"source": path.split("/")[-1], "plans": plans, "dram_bytes_per_plan": dram,
               "warp_inst_per_plan": sum(v["warp_inst_per_plan"] for v in kernels.values()),
               "kernels": kernels}
    json.dump(summary, open(f"{prefix}_launches_bench_summary.json", "w"), indent=1)
    top = {k: {f: round(v[f], 2) for f in ("share", "issue_active_pct", "threads_per_warp_inst", "fp64_pipe_pct")
               if f in v} for k, v in kernels.items() if v["share"] > 0.01}
    json.dump({"source": path.split("/")[-1], "kernels": top}, open(f"{prefix}_ncu_metrics.json", "w"), indent=1)
    for k, v in kernels.items():
        print(f"{k:40s} {v['launches']:4d} {v['ms']:9.2f} ms {100 * v['share']:5.1f}%  "
              f"{v['warp_inst_per_plan']:7.0f} inst/plan {v['dram_bytes_per_plan']:7.1f} B/plan  "
              f"issue {v.get('issue_active_pct', 0):5.1f}%  thr/warp {v.get('threads_per_warp_inst', 0):5.1f}  "
              f"fp64 {v.get('fp64_pipe_pct', 0):5.1f}%")
    print(f"total DRAM {dram:.1f} B/plan")


if __name__ == "__main__":
    main()
